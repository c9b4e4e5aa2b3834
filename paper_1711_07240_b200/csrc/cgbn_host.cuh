// cgbn_host.cuh — host-side planning, configuration choice and launches
// Part of the single translation unit cgbn.cu (included there, in order).

#pragma once

namespace {

// ----------------------------------------------------------------------------------
// Host-side planning

int num_sms_cached() {
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (cache[dev] == 0) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0)
      v = 148;
    cache[dev] = v;
  }
  return cache[dev];
}

int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// A/B switches and debug knobs, read once per process, never per launch.
struct Env {
  bool no_rows, no_masked, no_ct, no_pdl, ew_forward, ew_persistent, debug_plan;
  int rows_cs4 = 0;           // CGBN_ROWS_CS4
  int ct_tl = 0, ct_kc = 0;   // CGBN_CT_FORCE=tl,kc
  Env() {
    no_rows = getenv("CGBN_NO_ROWS") != nullptr;
    no_masked = getenv("CGBN_NO_MASKED") != nullptr;
    no_ct = getenv("CGBN_NO_CT") != nullptr;
    no_pdl = getenv("CGBN_NO_PDL") != nullptr;
    ew_forward = getenv("CGBN_EW_FORWARD") != nullptr;
    ew_persistent = getenv("CGBN_EW_PERSISTENT") != nullptr;
    debug_plan = getenv("CGBN_DEBUG_PLAN") != nullptr;
    if (const char* e = getenv("CGBN_ROWS_CS4")) rows_cs4 = atoi(e);
    if (const char* f = getenv("CGBN_CT_FORCE")) {
      if (sscanf(f, "%d,%d", &ct_tl, &ct_kc) != 2) ct_tl = ct_kc = 0;
    }
  }
};
const Env& env() {
  static const Env e;
  return e;
}

// Workspace: tickets + barrier words | (C + max grid) double2 per-CTA partial slots |
// coefficient table (5 x C doubles: P, Q, A, B, Cc).
// Row reductions (NHWC / 2-D, C % 4 == 0): rows per block >= 32 keeps the partial
// slots (nb * C double2) under 1/8 of the activation bytes.
bool rows_layout(int64_t C, int64_t HW, int layout) {
  return (layout == CGBN_LAYOUT_NHWC || HW == 1) && C % 4 == 0 && !env().no_rows;
}

NGeom rows_geom(int64_t N, int64_t C, int64_t HW, int64_t ctas) {
  NGeom g;
  g.M = (uint32_t)(N * HW);
  g.C = (uint32_t)C;
  g.C4 = (uint32_t)(C / 4);
  // Channel slice width in float4 units. Narrow slices put more rows in flight per CTA
  // (rpp = 256 / CS4) for the same slot table (nb * C = ctas * 4 * CS4 partials), which
  // is what wide-C layers lacked: measured on B200 in a graph (tools/rows_sweep.sh),
  // 128 channels per slice (CS4 = 32) is best up to C = 256 and on tiny row counts, 256
  // channels (CS4 = 64) above that; full-width 1024-channel slices were 10-70% slower
  // on C >= 512 (e.g. [32,2048,7,7] stats 10.1 -> 7.4 us, bwd reduce 14.6 -> 9.2 us).
  uint32_t cs_max = (g.C4 > 64 && g.M >= 256) ? 64u : 32u;
  const int v = env().rows_cs4;  // A/B
  if (v == 32 || v == 64 || v == 128 || v == 256) cs_max = (uint32_t)v;
  g.CS4 = g.C4 < cs_max ? g.C4 : cs_max;
  g.rpp = (uint32_t)kThreads / g.CS4;
  g.nslices = (g.C4 + g.CS4 - 1) / g.CS4;
  int64_t nb = ceil_div(ctas, (int64_t)g.nslices);
  const int64_t cap = (int64_t)g.M / 32;
  if (nb > cap) nb = cap;
  if (nb > (int64_t)g.M) nb = g.M;
  g.nb = (uint32_t)(nb < 1 ? 1 : nb);
  return g;
}

size_t slots_bytes(int64_t N, int64_t C, int64_t HW, int layout, int sms) {
  size_t n = (size_t)C + (size_t)sms * kMaxCtasPerSm;
  if (rows_layout(C, HW, layout)) {
    const NGeom g = rows_geom(N, C, HW, (int64_t)sms * kMaxCtasPerSm);
    const size_t r = (size_t)g.nb * (size_t)C;
    if (r > n) n = r;
  }
  return n * sizeof(double2);
}
size_t ws_bytes_for(int64_t N, int64_t C, int64_t HW, int layout, int sms) {
  // coefficients: P, Q, A, B, Cc (fp64), then the fp32 records T1 (float4) and T2 (float2)
  return kTicketBytes + slots_bytes(N, C, HW, layout, sms) + (8 * (size_t)C + 2) * sizeof(double);
}

struct WsView {
  unsigned* tickets;
  unsigned* bar;
  double2* slots;
  double* P;
  double* Q;
  double* A;
  double* B;
  double* Cc;
  float4* T1;  // fp32 records of the 16-bit elementwise passes (cgbn_ops.cuh)
  float2* T2;
};

int ws_view(void* ws, size_t ws_bytes, int64_t N, int64_t C, int64_t HW, int layout,
            WsView* v) {
  const int sms = num_sms_cached();
  const size_t need = ws_bytes_for(N, C, HW, layout, sms);
  if (!ws || ws_bytes < need)
    return set_error(CGBN_ERR_INVALID, "workspace too small: need %zu bytes, got %zu", need,
                     ws_bytes);
  if (reinterpret_cast<uintptr_t>(ws) % 16)
    return set_error(CGBN_ERR_INVALID, "workspace must be 16-byte aligned");
  char* b = reinterpret_cast<char*>(ws);
  v->tickets = reinterpret_cast<unsigned*>(b);
  v->bar = v->tickets + kTicketWords;
  v->slots = reinterpret_cast<double2*>(b + kTicketBytes);
  double* coef =
      reinterpret_cast<double*>(b + kTicketBytes + slots_bytes(N, C, HW, layout, sms));
  v->P = coef;
  v->Q = coef + C;
  v->A = coef + 2 * C;
  v->B = coef + 3 * C;
  v->Cc = coef + 4 * C;
  v->T1 = reinterpret_cast<float4*>(coef + ((5 * C + 1) & ~(int64_t)1));  // 16-byte aligned
  v->T2 = reinterpret_cast<float2*>(reinterpret_cast<double*>(v->T1) + 2 * C);
  return CGBN_OK;
}

// Per-(kernel, device) caches. Keyed by the kernel's address: kernels of one signature
// share a function-pointer type, so a per-template static would alias them.
std::mutex g_cache_mu;
std::map<std::pair<const void*, int>, int> g_occ_cache;
std::map<std::pair<const void*, int>, bool> g_smem_done;

template <class K>
int64_t resident_ctas(K kernel) {
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_pair(reinterpret_cast<const void*>(kernel), dev);
  int occ = 0;
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    auto it = g_occ_cache.find(key);
    if (it != g_occ_cache.end()) occ = it->second;
  }
  if (occ == 0) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kThreads, 0) != cudaSuccess ||
        occ <= 0)
      occ = 1;
    if (occ > kMaxCtasPerSm) occ = kMaxCtasPerSm;
    std::lock_guard<std::mutex> lk(g_cache_mu);
    g_occ_cache[key] = occ;
  }
  return (int64_t)num_sms_cached() * occ;
}

template <class K>
void smem_optin(K kernel, size_t smem_bytes) {
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_pair(reinterpret_cast<const void*>(kernel), dev);
  std::lock_guard<std::mutex> lk(g_cache_mu);
  if (g_smem_done.count(key)) return;
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes);
  g_smem_done[key] = true;
}

// The ABI's `layout` argument carries the activation dtype in bits 4..7
// (CGBN_ACT_F32 / CGBN_ACT_BF16 / CGBN_ACT_F16, include/cgbn.h).
int split_fmt(int* layout, int* act) {
  const int f = *layout;
  *act = (f >> 4) & 0xF;
  *layout = f & 0xF;
  if (f & ~0xFF) return set_error(CGBN_ERR_INVALID, "unknown layout/format bits 0x%x", f);
  if (*act > 2) return set_error(CGBN_ERR_INVALID, "unknown activation dtype %d", *act);
  return CGBN_OK;
}

int act_bytes(int act) { return act == 0 ? 4 : 2; }

int validate_shape(int64_t N, int64_t C, int64_t HW, int layout) {
  if (N < 1 || C < 1 || HW < 1)
    return set_error(CGBN_ERR_INVALID, "extents must be positive, got N=%lld C=%lld HW=%lld",
                     (long long)N, (long long)C, (long long)HW);
  if (layout != CGBN_LAYOUT_NCHW && layout != CGBN_LAYOUT_NHWC)
    return set_error(CGBN_ERR_INVALID, "unknown layout %d", layout);
  if (C > 65535) return set_error(CGBN_ERR_INVALID, "C=%lld exceeds 65535", (long long)C);
  if (N * HW >= (1ll << 31))
    return set_error(CGBN_ERR_INVALID, "per-channel count N*HW=%lld must be < 2^31",
                     (long long)(N * HW));
  if (N * C * HW >= (1ll << 32))
    return set_error(CGBN_ERR_INVALID, "tensor of %lld elements exceeds 2^32",
                     (long long)(N * C * HW));
  return CGBN_OK;
}

struct Plan {
  int act;  // activation dtype (0 fp32, 1 bf16, 2 fp16)
  int vec;
  bool rows;  // NHWC / 2-D with C % 4 == 0: row reduction (k_reduce_rows + k_fold_rows)
  bool team;
  bool ct;   // NCHW: cluster-team reduction (k_reduce_ct) when it fills the GPU
  Geom g;
  int64_t elems;
};

// Reduction plan. `ptrs` are every activation pointer the kernel touches; the vector
// width is the widest one that divides the plane length and the alignment of all.
int make_plan(int64_t N, int64_t C, int64_t HW, int layout, int act, const void* const* ptrs,
              int nptr, Plan* out) {
  int rc = validate_shape(N, C, HW, layout);
  if (rc) return rc;
  int64_t planeN = N, planeHW = HW;
  if (layout == CGBN_LAYOUT_NHWC) { planeN = N * HW; planeHW = 1; }
  uintptr_t align = 0;
  for (int k = 0; k < nptr; ++k) align |= (uintptr_t)ptrs[k];
  const int es = act_bytes(act);
  const int64_t vmax = 16 / es;  // elements per 16-byte unit
  const int64_t E = N * C * HW;
  int vec = 1;
  if (planeHW % vmax == 0 && (align % 16) == 0) vec = (int)vmax;
  else if (es == 2 && planeHW % 4 == 0 && (align % 8) == 0)
    vec = 4;  // exact 8-byte units: faster than masked 16-byte covers (bf16 14x14 stats 4.4 -> 3.3 us)
  else if (layout == CGBN_LAYOUT_NCHW && HW >= 16 && (align % 16) == 0 && E % vmax == 0 &&
           E + 2 * vmax < (1ll << 32) && !env().no_masked)
    vec = es == 4 ? 5 : 9;  // masked 16-byte cover of odd planes (never leaves the tensor)
  else if (es == 2 && planeHW % 4 == 0 && (align % 8) == 0) vec = 4;
  else if (planeHW % 2 == 0 && (align % (2 * es)) == 0) vec = 2;
  const int V = vec_of(vec);
  Geom g;
  g.C = (uint32_t)C;
  g.HW = (uint32_t)planeHW;
  g.HWv = (uint32_t)(masked_vm(vec) ? (planeHW + V - 1) / V + 1 : planeHW / vec);
  g.Lv = (uint32_t)(planeN * g.HWv);
  g.gap = (uint64_t)(C - 1) * g.HWv;
  g.dhw.init(g.HWv);
  g.count = (double)(N * HW);
  g.T = (uint64_t)C * g.Lv;
  g.grid = 1;
  // team size: smallest power of two in [32, 256] giving <= ~8 units per thread
  uint32_t tl = 5;
  while (tl < 8 && (((uint64_t)g.Lv + (1ull << tl) - 1) >> tl) > 8) ++tl;
  g.tpc_log2 = tl;
  out->act = act;
  out->vec = vec;
  out->team = g.Lv <= kTeamMaxLv;
  out->ct = layout == CGBN_LAYOUT_NCHW && !env().no_ct;
  out->rows = rows_layout(C, HW, layout) && (align % 16) == 0;
  out->g = g;
  out->elems = N * C * HW;
  return CGBN_OK;
}

int fill_parts(Parts* P, const double* const* partials, int G) {
  if (G < 1 || G > CGBN_MAX_GROUP)
    return set_error(CGBN_ERR_INVALID, "group size %d outside [1, %d]", G, CGBN_MAX_GROUP);
  if (!partials) return set_error(CGBN_ERR_INVALID, "partials array is NULL");
  for (int r = 0; r < G; ++r) {
    if (!partials[r]) return set_error(CGBN_ERR_INVALID, "partials[%d] is NULL", r);
    P->p[r] = partials[r];
  }
  for (int r = G; r < CGBN_MAX_GROUP; ++r) P->p[r] = nullptr;
  P->G = G;
  return CGBN_OK;
}

template <class K>
unsigned flat_grid(K kernel, const Plan& pl) {
  int64_t grid = resident_ctas(kernel);
  const int64_t want = ceil_div(pl.elems, kMinElemsPerCta);
  if (want < grid) grid = want;
  return (unsigned)(grid < 1 ? 1 : grid);
}

template <class K>
unsigned team_grid(K kernel, const Plan& pl) {
  const int64_t cpt = kThreads >> pl.g.tpc_log2;
  int64_t grid = ceil_div(pl.g.C, cpt);
  const int64_t res = resident_ctas(kernel);
  if (grid > res) grid = res;
  return (unsigned)(grid < 1 ? 1 : grid);
}

// Launch with programmatic dependent launch allowed (see pdl_trigger / pdl_wait).
bool pdl_enabled() { return !env().no_pdl; }

template <class K, class... Args>
void launch_pdl(K kernel, unsigned grid, bool pdl, cudaStream_t st, Args... args) {
  if (!pdl || !pdl_enabled()) {
    kernel<<<grid, kThreads, 0, st>>>(args...);
    return;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, args...);
}

// Clusters of `kc` CTAs of `kernel` that can be co-resident (cached; 0 if unsupported).
std::map<std::tuple<const void*, int, int>, int> g_cluster_cache;

template <class K>
int64_t cluster_capacity(K kernel, uint32_t kc) {
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_tuple(reinterpret_cast<const void*>(kernel), dev, (int)kc);
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    auto it = g_cluster_cache.find(key);
    if (it != g_cluster_cache.end()) return (int64_t)it->second * kc;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(kc * 64);
  cfg.blockDim = dim3(kThreads);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = kc;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kernel, &cfg) != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  std::lock_guard<std::mutex> lk(g_cache_mu);
  g_cluster_cache[key] = n;
  return (int64_t)n * kc;
}

struct CtCfg {
  int tl;
  uint32_t kc, grid;
};

// Cluster-team configuration, from the lab sweep (tools/flatlab.cu "sweep", B200,
// ResNet-50 shapes). Cluster sizes are powers of two; U = vector loads of each input a
// thread keeps in flight per round.
//  - latency-bound (the whole stream fits in one round of the resident slots): the
//    fewest CTAs whose threads need a single round, unclustered first (a cluster costs
//    ~1 us of barrier + DSMEM at these sizes);
//  - bandwidth-bound: the largest grid that fits in one wave (bytes in flight), then the
//    smaller cluster, then the larger team.
// Returns false when nothing fills a quarter of the slots (tiny C: the flat kernel
// spreads one channel over more CTAs than a cluster holds).
template <class Op>
int64_t ct_cluster_cap(int tl, uint32_t kc) {
  switch (tl) {
    case 8: return cluster_capacity(k_reduce_ct<Op, 8>, kc);
    case 7: return cluster_capacity(k_reduce_ct<Op, 7>, kc);
    case 6: return cluster_capacity(k_reduce_ct<Op, 6>, kc);
    default: return cluster_capacity(k_reduce_ct<Op, 5>, kc);
  }
}

template <class Op>
bool choose_ct(const Plan& pl, CtCfg* cfg) {
  constexpr int64_t U = unroll_for<Op::kVec, Op::kIn>();
  const int64_t slots = resident_ctas(k_reduce_ct<Op, 8>);
  const int64_t C = pl.g.C, Lv = pl.g.Lv;
  bool latency_bound = C * Lv <= slots * kThreads * U;
  int64_t best_n = 0;
  double best = 1e30;
again:
  for (uint32_t kc = 1; kc <= 8; kc *= 2) {
    for (int tl = 8; tl >= 5; --tl) {
      const int64_t tpc = 1 << tl;
      if (kc > 1 && Lv / kc < tpc) continue;  // every thread keeps >= 1 unit
      const int64_t n = ceil_div(C, (int64_t)kThreads >> tl) * kc;
      if (n > slots) continue;
      const int64_t units = ceil_div(Lv, (int64_t)kc * tpc);
      double score;
      if (latency_bound) {
        if (units > U) continue;
        score = (kc > 1 ? 1e6 : 0.0) + (double)n;  // unclustered, then fewest CTAs
      } else {
        score = -(double)n * 16.0 + kc;  // most CTAs, then smallest cluster
      }
      if (score >= best) continue;
      if (kc > 1 && n > ct_cluster_cap<Op>(tl, kc)) continue;
      best = score;
      best_n = n;
      cfg->tl = tl;
      cfg->kc = kc;
      cfg->grid = (uint32_t)n;
    }
  }
  if (latency_bound && best_n == 0) {
    latency_bound = false;  // no single-round configuration: rank by fill instead
    goto again;
  }
  {  // CGBN_CT_FORCE=tl,kc (experiments only)
    const int tl = env().ct_tl, kc = env().ct_kc;
    if (tl >= 5 && tl <= 8 && kc >= 1 && kc <= 8) {
      cfg->tl = tl;
      cfg->kc = (uint32_t)kc;
      cfg->grid = (uint32_t)(ceil_div(C, (int64_t)kThreads >> tl) * kc);
      best_n = cfg->grid;
    }
  }
  if (env().debug_plan)
    fprintf(stderr, "[cgbn] ct C=%lld Lv=%lld in=%d slots=%lld %s -> tl=%d kc=%u grid=%lld\n",
            (long long)C, (long long)Lv, Op::kIn, (long long)slots,
            latency_bound ? "latency" : "bandwidth", best_n ? cfg->tl : -1, best_n ? cfg->kc : 0,
            (long long)best_n);
  if (best_n == 0 && ceil_div(C, kThreads >> 5) > slots) {
    // very wide layers: 8 channels per CTA, CTAs loop over channel groups
    cfg->tl = 5;
    cfg->kc = 1;
    cfg->grid = (uint32_t)slots;
    return true;
  }
  return best_n * 4 >= slots;
}

template <class Op, int TL>
int launch_ct(Geom g, const Op& op, double* out, uint32_t kc, cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(g.grid);
  cfg.blockDim = dim3(kThreads);
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  int na = 0;
  if (kc > 1) {
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = kc;
    at[na].val.clusterDim.y = 1;
    at[na].val.clusterDim.z = 1;
    ++na;
  }
  if (pdl_enabled()) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, k_reduce_ct<Op, TL>, g, op, out);
  if (e != cudaSuccess)
    return set_error(CGBN_ERR_CUDA, "cluster reduction launch failed: %s", cudaGetErrorString(e));
  return CGBN_OK;
}

template <class Op>
int launch_reduce(const Plan& pl, const Op& op, double* out, const WsView& w, cudaStream_t st) {
  Geom g = pl.g;
  CtCfg cc;
  if (pl.ct && choose_ct<Op>(pl, &cc)) {
    g.grid = cc.grid;
    switch (cc.tl) {
      case 8: return launch_ct<Op, 8>(g, op, out, cc.kc, st);
      case 7: return launch_ct<Op, 7>(g, op, out, cc.kc, st);
      case 6: return launch_ct<Op, 6>(g, op, out, cc.kc, st);
      default: return launch_ct<Op, 5>(g, op, out, cc.kc, st);
    }
  }
  if (pl.team) {
    g.grid = team_grid(k_reduce_team<Op>, pl);
    launch_pdl(k_reduce_team<Op>, g.grid, true, st, g, op, out);
  } else {
    g.grid = flat_grid(k_reduce_flat<Op>, pl);
    launch_pdl(k_reduce_flat<Op>, g.grid, true, st, g, op, out, w.slots, w.tickets);
  }
  return CGBN_OK;
}

// Row reduction (NHWC / 2-D): k_reduce_rows -> k_fold_rows (finisher of `op`).
template <class NOp, class Op>
int launch_rows(const Plan& pl, const NOp& nop, const Op& op, double* out, const WsView& w,
                cudaStream_t st) {
  const int64_t N = 1, HW = pl.g.count;  // rows = N*HW of the original geometry
  const NGeom ng = rows_geom(N, pl.g.C, HW, resident_ctas(k_reduce_rows<NOp>));
  const unsigned grid = ng.nslices * ng.nb;
  launch_pdl(k_reduce_rows<NOp>, grid, true, st, ng, nop, w.slots);
  Geom g = pl.g;
  const unsigned fgrid = (unsigned)ceil_div((int64_t)pl.g.C * 32, kThreads);
  launch_pdl(k_fold_rows<Op>, fgrid, true, st, g, op, (const double2*)w.slots, ng.nb, out);
  return CGBN_OK;
}

// The fused-exchange push of the *_p2p entry points (thread-local: set around one
// dispatch by the calling thread; every other call reduces into `out`).
thread_local const p2p::Push* g_push = nullptr;


// Forward statistics in mode kPartial / kRawSums / kLocalFinal / kSumSq (PUSH: the
// kPartial finisher pushes into the fused exchange's regions instead of `out`).
template <class T, int VEC, bool PUSH>
int run_stats_op(const Plan& pl, const T* x, bool shift, int mode, double* out, double* out2,
                 const FwdFinal* F, const WsView& w, cudaStream_t st, const double* ksum,
                 const double* kcount) {
  StatsOp<T, VEC, PUSH> op;
  op.x = x;
  op.K = 0.0;
  op.shift = shift;
  op.ksum = ksum;
  op.kcount = kcount;
  op.mode = mode;
  op.out2 = out2;
  if constexpr (PUSH) op.push = *g_push;
  if (F) op.F = *F;
  if constexpr (VEC == 1) {
    if (pl.rows) {
      StatsRows<T, PUSH> nop;
      nop.base = op;
      nop.gg = pl.g;
      return launch_rows(pl, nop, op, out, w, st);
    }
  }
  return launch_reduce(pl, op, out, w, st);
}

template <class T, int VEC>
int run_stats(const Plan& pl, const void* xv, bool shift, int mode, double* out, double* out2,
              const FwdFinal* F, const WsView& w, cudaStream_t st, const double* ksum,
              const double* kcount) {
  const T* x = static_cast<const T*>(xv);
  if (g_push && mode == kPartial)
    return run_stats_op<T, VEC, true>(pl, x, shift, mode, out, out2, F, w, st, ksum, kcount);
  return run_stats_op<T, VEC, false>(pl, x, shift, mode, out, out2, F, w, st, ksum, kcount);
}

template <class T, int VEC, bool RELU, bool PUSH>
int run_bwd_op(const Plan& pl, const T* dy, const T* x, const double* saved, const float* gamma,
               const float* beta, int mode, double* out, const BwdFinal* F, const WsView& w,
               cudaStream_t st) {
  BwdOp<T, VEC, RELU, PUSH> op;
  op.dy = dy;
  op.x = x;
  op.saved = saved;
  op.gamma = gamma;
  op.beta = beta;
  op.mean = op.P = op.Q = 0.0;
  op.mode = mode;
  if constexpr (PUSH) op.push = *g_push;
  if (F) op.F = *F;
  if constexpr (VEC == 1) {
    if (pl.rows) {
      BwdRows<T, RELU, PUSH> nop;
      nop.base = op;
      nop.gg = pl.g;
      return launch_rows(pl, nop, op, out, w, st);
    }
  }
  return launch_reduce(pl, op, out, w, st);
}

template <class T, int VEC, bool RELU>
int run_bwd_reduce(const Plan& pl, const void* dyv, const void* xv, const double* saved,
                   const float* gamma, const float* beta, int mode, double* out,
                   const BwdFinal* F, const WsView& w, cudaStream_t st) {
  const T* dy = static_cast<const T*>(dyv);
  const T* x = static_cast<const T*>(xv);
  if (g_push && mode == kPartial)
    return run_bwd_op<T, VEC, RELU, true>(pl, dy, x, saved, gamma, beta, mode, out, F, w, st);
  return run_bwd_op<T, VEC, RELU, false>(pl, dy, x, saved, gamma, beta, mode, out, F, w, st);
}

// fp32: vector modes 1, 2, 4, 5 (masked float4); bf16 / fp16: 1, 2, 4, 8, 9 (masked 8).
template <class T>
int dispatch_stats_t(const Plan& pl, const void* x, bool shift, int mode, double* out,
                     double* out2, const FwdFinal* F, const WsView& w, cudaStream_t st,
                     const double* ksum, const double* kcount) {
  if constexpr (sizeof(T) == 4) {
    switch (pl.vec) {
      case 5: return run_stats<T, 5>(pl, x, shift, mode, out, out2, F, w, st, ksum, kcount);
      case 4: return run_stats<T, 4>(pl, x, shift, mode, out, out2, F, w, st, ksum, kcount);
      case 2: return run_stats<T, 2>(pl, x, shift, mode, out, out2, F, w, st, ksum, kcount);
      default: return run_stats<T, 1>(pl, x, shift, mode, out, out2, F, w, st, ksum, kcount);
    }
  } else {
    switch (pl.vec) {
      case 9: return run_stats<T, 9>(pl, x, shift, mode, out, out2, F, w, st, ksum, kcount);
      case 8: return run_stats<T, 8>(pl, x, shift, mode, out, out2, F, w, st, ksum, kcount);
      case 4: return run_stats<T, 4>(pl, x, shift, mode, out, out2, F, w, st, ksum, kcount);
      case 2: return run_stats<T, 2>(pl, x, shift, mode, out, out2, F, w, st, ksum, kcount);
      default: return run_stats<T, 1>(pl, x, shift, mode, out, out2, F, w, st, ksum, kcount);
    }
  }
}

int dispatch_stats(const Plan& pl, const void* x, bool shift, int mode, double* out,
                   double* out2, const FwdFinal* F, const WsView& w, cudaStream_t st,
                   const double* ksum = nullptr, const double* kcount = nullptr) {
  CGBN_ROUTED(pl.act);
  return dispatch_stats_t<TuAct>(pl, x, shift, mode, out, out2, F, w, st, ksum, kcount);
}

template <class T, bool RELU>
int dispatch_bwd_t(const Plan& pl, const void* dy, const void* x, const double* saved,
                   const float* gamma, const float* beta, int mode, double* out,
                   const BwdFinal* F, const WsView& w, cudaStream_t st) {
  if constexpr (sizeof(T) == 4) {
    switch (pl.vec) {
      case 5: return run_bwd_reduce<T, 5, RELU>(pl, dy, x, saved, gamma, beta, mode, out, F, w, st);
      case 4: return run_bwd_reduce<T, 4, RELU>(pl, dy, x, saved, gamma, beta, mode, out, F, w, st);
      case 2: return run_bwd_reduce<T, 2, RELU>(pl, dy, x, saved, gamma, beta, mode, out, F, w, st);
      default:
        return run_bwd_reduce<T, 1, RELU>(pl, dy, x, saved, gamma, beta, mode, out, F, w, st);
    }
  } else {
    switch (pl.vec) {
      case 9: return run_bwd_reduce<T, 9, RELU>(pl, dy, x, saved, gamma, beta, mode, out, F, w, st);
      case 8: return run_bwd_reduce<T, 8, RELU>(pl, dy, x, saved, gamma, beta, mode, out, F, w, st);
      case 4: return run_bwd_reduce<T, 4, RELU>(pl, dy, x, saved, gamma, beta, mode, out, F, w, st);
      case 2: return run_bwd_reduce<T, 2, RELU>(pl, dy, x, saved, gamma, beta, mode, out, F, w, st);
      default:
        return run_bwd_reduce<T, 1, RELU>(pl, dy, x, saved, gamma, beta, mode, out, F, w, st);
    }
  }
}

template <class T>
int dispatch_bwd_r(const Plan& pl, const void* dy, const void* x, const double* saved,
                   const float* gamma, const float* beta, bool relu, int mode, double* out,
                   const BwdFinal* F, const WsView& w, cudaStream_t st) {
  return relu ? dispatch_bwd_t<T, true>(pl, dy, x, saved, gamma, beta, mode, out, F, w, st)
              : dispatch_bwd_t<T, false>(pl, dy, x, saved, gamma, beta, mode, out, F, w, st);
}

int dispatch_bwd_reduce(const Plan& pl, const void* dy, const void* x, const double* saved,
                        const float* gamma, const float* beta, bool relu, int mode, double* out,
                        const BwdFinal* F, const WsView& w, cudaStream_t st) {
  CGBN_ROUTED(pl.act);
  return dispatch_bwd_r<TuAct>(pl, dy, x, saved, gamma, beta, relu, mode, out, F, w, st);
}

// ---- elementwise

struct EwPlan {
  EwGeom g;
  int cm;
  int act;
};

int make_ew(int64_t N, int64_t C, int64_t HW, int layout, int act, const void* const* ptrs,
            int nptr, EwPlan* out) {
  int rc = validate_shape(N, C, HW, layout);
  if (rc) return rc;
  uintptr_t align = 0;
  for (int k = 0; k < nptr; ++k) align |= (uintptr_t)ptrs[k];
  if (align % 16)
    return set_error(CGBN_ERR_INVALID, "activation pointers must be 16-byte aligned");
  const uint64_t E = (uint64_t)N * C * HW;
  const uint32_t UE = 16 / act_bytes(act);  // elements per 16-byte unit
  EwGeom& g = out->g;
  g.C = (uint32_t)C;
  g.HW = (uint32_t)HW;
  g.n4 = (uint32_t)(E / UE);
  g.tail = (uint32_t)(E % UE);
  g.dhw.init((uint32_t)HW);
  g.dc.init((uint32_t)C);
  // Sweep from the end of the tensor: the preceding channel-major reduction read the
  // high-n planes of every channel last, so they are the likeliest L2 hits (measured
  // +1.5% on the ResNet-50 step, up to 7% on the 100 MB layers; CGBN_EW_FORWARD=1 off).
  g.rev = env().ew_forward ? 0u : 1u;
  g.reuse = 0;
  // channel modes work on 4-element chunks of a unit: CM 0 / 3 need HW % 4 / C % 4 only
  (void)UE;
  if (layout == CGBN_LAYOUT_NHWC || HW == 1) out->cm = (C % 4 == 0) ? 3 : 2;
  else out->cm = (HW % 4 == 0) ? 0 : 1;
  out->act = act;
  return CGBN_OK;
}

// One round of kEwU units per thread, not a persistent grid: a copy-like kernel streams
// faster with many short-lived CTAs than with one resident wave that loops (ResNet-50
// step +3%, 100 MB layers 4-6 us faster; CGBN_EW_PERSISTENT=1 restores the resident
// grid for A/B).
// Units per thread per round: kEwU (2) in memory order; channels_last (CM 3) threads
// keep their UE channels' fp64 coefficients in registers, so they take more units to
// amortise the coefficient loads.
// Measured on B200 (U = 1 / 2 / 4 / 8, [32,C,H,W] NHWC): 4 is best everywhere except the
// fp32 dx pass without ReLU, where 8 is (54 -> 48 us on [32,256,56,56]), and the 16-bit
// dx pass with ReLU: its five 8-wide coefficient tables take ~160 registers, so one CTA
// per SM runs and only more units in flight hide the latency (U = 1 / 2 / 4 / 8: 170 /
// 111 / 79 / 62 us). 16-bit dx without ReLU at 8 (40 -> 50 us) and fp32 dx with ReLU at 8
// are slower.
#ifndef CGBN_EWU_NHWC
#define CGBN_EWU_NHWC 4
#endif
#ifndef CGBN_EWU_NHWC_RELU16
#define CGBN_EWU_NHWC_RELU16 8
#endif
template <int CM, class T = float, bool DX = false, bool RELU = false>
constexpr int ew_units() {
  return CM != 3                               ? kEwU
         : (DX && !RELU && sizeof(T) == 4)     ? 2 * CGBN_EWU_NHWC
         : (DX && RELU && sizeof(T) == 2)      ? CGBN_EWU_NHWC_RELU16
                                               : CGBN_EWU_NHWC;
}

template <class K>
unsigned ew_grid(K kernel, const EwPlan& ep, int units = kEwU) {
  int64_t grid = ceil_div((int64_t)ep.g.n4 + 1, kThreads * units);
  if (env().ew_persistent) {
    const int64_t res = resident_ctas(kernel);
    if (grid > res) grid = res;
  }
  return (unsigned)(grid < 1 ? 1 : grid);
}

// pdl: the kernel before this launch on `st` is one of ours that does not write x
// (a reduction, finalize or coefficient kernel), so x may be prefetched before the
// dependency wait.
// Grid plus the channels_last coefficient-reuse flag (a thread's units are gridDim*256
// units apart; they share their channels when that distance covers whole rows).
template <class K>
unsigned ew_grid_geom(K kernel, const EwPlan& ep, EwGeom* g, int units) {
  unsigned grid = ew_grid(kernel, ep, units);
  *g = ep.g;
  const uint64_t ue = ep.act == 0 ? 4 : 8;
  if (ep.cm == 3 && ep.g.C > 0) {
    // round the grid up to the channel period when that idles few CTAs: e.g. fp32
    // C = 2048 needs an even grid, and [32,2048,7,7] had an odd one (785), so every
    // unit reloaded its fp64 coefficients (normalise 11.2 us vs 7.8 us NCHW)
    const uint64_t per = ue * kThreads;
    uint64_t a = ep.g.C, b = per;
    while (b) { const uint64_t t = a % b; a = b; b = t; }
    const uint64_t m = ep.g.C / a;
    const uint64_t up = (grid + m - 1) / m * m;
    if (up - grid <= grid / 8) grid = (unsigned)up;
  }
  g->reuse = (ep.cm == 3 && (ue * (uint64_t)grid * kThreads) % ep.g.C == 0) ? 1u : 0u;
  return grid;
}

template <class T, bool RELU, int CM>
void launch_ew_affine_t(const EwPlan& ep, const void* x, void* y, const double* P,
                        const double* Q, const float4* T1, bool pdl, cudaStream_t st) {
  EwGeom g;
  constexpr int U = ew_units<CM>();
  const unsigned grid = ew_grid_geom(k_ew_affine<T, RELU, CM, U>, ep, &g, U);
  launch_pdl(k_ew_affine<T, RELU, CM, U>, grid, pdl, st, g, static_cast<const T*>(x),
             static_cast<T*>(y), P, Q, T1);
}

template <class T, bool RELU>
void launch_ew_affine_r(const EwPlan& ep, int cm, const void* x, void* y, const double* P,
                        const double* Q, const float4* T1, bool pdl, cudaStream_t st) {
  if (cm == 0) launch_ew_affine_t<T, RELU, 0>(ep, x, y, P, Q, T1, pdl, st);
  else if (cm == 1) launch_ew_affine_t<T, RELU, 1>(ep, x, y, P, Q, T1, pdl, st);
  else if (cm == 2) launch_ew_affine_t<T, RELU, 2>(ep, x, y, P, Q, T1, pdl, st);
  else launch_ew_affine_t<T, RELU, 3>(ep, x, y, P, Q, T1, pdl, st);
}

template <class T>
void launch_ew_affine_d(const EwPlan& ep, int cm, bool relu, const void* x, void* y,
                        const double* P, const double* Q, const float4* T1, bool pdl,
                        cudaStream_t st) {
  if (relu) launch_ew_affine_r<T, true>(ep, cm, x, y, P, Q, T1, pdl, st);
  else launch_ew_affine_r<T, false>(ep, cm, x, y, P, Q, T1, pdl, st);
}

// T1: the forward finisher's fp32 records (16-bit activations, no ReLU: the fp32 path of
// k_ew_affine), or null for caller-provided tables (eval, x_hat, channel_affine).
void launch_ew_affine(const EwPlan& ep, bool relu, const void* x, void* y, const double* P,
                      const double* Q, cudaStream_t st, bool pdl = true,
                      const float4* T1 = nullptr) {
  int cm = ep.cm;
  if (cm == 3 && (((uintptr_t)P | (uintptr_t)Q) % 16) != 0) cm = 2;  // caller's tables
  launch_ew_affine_d<TuAct>(ep, cm, relu, x, y, P, Q, T1, pdl, st);
}

template <class T, bool RELU, int CM>
void launch_ew_dx_t(const EwPlan& ep, const void* dy, const void* x, void* dx, const WsView& w,
                    cudaStream_t st) {
  EwGeom g;
  constexpr int U = ew_units<CM, T, true, RELU>();
  const unsigned grid = ew_grid_geom(k_ew_dx<T, RELU, CM, U>, ep, &g, U);
  launch_pdl(k_ew_dx<T, RELU, CM, U>, grid, true, st, g,
             static_cast<const T*>(dy), static_cast<const T*>(x), static_cast<T*>(dx),
             (const double*)w.A, (const double*)w.B, (const double*)w.Cc, (const double*)w.P,
             (const double*)w.Q, (const float4*)w.T1, (const float2*)w.T2);
}

template <class T, bool RELU>
void launch_ew_dx_r(const EwPlan& ep, const void* dy, const void* x, void* dx, const WsView& w,
                    cudaStream_t st) {
  if (ep.cm == 0) launch_ew_dx_t<T, RELU, 0>(ep, dy, x, dx, w, st);
  else if (ep.cm == 1) launch_ew_dx_t<T, RELU, 1>(ep, dy, x, dx, w, st);
  else if (ep.cm == 2) launch_ew_dx_t<T, RELU, 2>(ep, dy, x, dx, w, st);
  else launch_ew_dx_t<T, RELU, 3>(ep, dy, x, dx, w, st);
}

template <class T>
void launch_ew_dx_d(const EwPlan& ep, bool relu, const void* dy, const void* x, void* dx,
                    const WsView& w, cudaStream_t st) {
  if (relu) launch_ew_dx_r<T, true>(ep, dy, x, dx, w, st);
  else launch_ew_dx_r<T, false>(ep, dy, x, dx, w, st);
}

void launch_ew_dx(const EwPlan& ep, bool relu, const void* dy, const void* x, void* dx,
                  const WsView& w, cudaStream_t st) {
  launch_ew_dx_d<TuAct>(ep, relu, dy, x, dx, w, st);
}

unsigned chan_blocks(int64_t C) { return (unsigned)ceil_div(C, 256); }

FwdFinal make_fwd_final(int64_t C, const float* gamma, const float* beta, double eps,
                        double momentum, float* rm, float* rv, double* saved, unsigned* status,
                        const WsView& w) {
  FwdFinal F;
  F.gamma = gamma; F.beta = beta;
  F.eps = eps; F.momentum = momentum;
  F.rmean = rm; F.rvar = rv;
  F.saved = saved;
  F.P = w.P; F.Q = w.Q;
  F.T1 = w.T1;
  F.status = status;
  F.C = (uint32_t)C;
  return F;
}

BwdFinal make_bwd_final(int64_t C, const double* saved, const float* gamma, const float* beta,
                        double eps, bool relu, float* dgamma, float* dbeta, unsigned* status,
                        const WsView& w) {
  BwdFinal F;
  F.saved = saved; F.gamma = gamma; F.beta = beta;
  F.eps = eps;
  F.relu = relu ? 1 : 0;
  F.A = w.A; F.B = w.B; F.Cc = w.Cc; F.P = w.P; F.Q = w.Q;
  F.T1 = w.T1; F.T2 = w.T2;
  F.dgamma = dgamma; F.dbeta = dbeta;
  F.status = status;
  F.C = (uint32_t)C;
  return F;
}

// ---- single-launch on-chip passes (cgbn_onchip.cuh), single-rank groups

// CGBN_NO_ONCHIP=1: always the split path (A/B). CGBN_ONCHIP_MAX_FRAC: the largest
// activation footprint (x, or dy + x) sent on chip, as a fraction of the GPU's total
// shared memory. Default from the in-step A/B on B200 (tools/gpu/onchip_frac.sh,
// profiles/r2_onchip_frac.jsonl; ResNet-50 b32 step, fp32):
//   0 (off) 2.118 ms, 0.1 2.114, 0.2 2.103, 0.4 2.088 (best), 0.8 2.344 ms.
// Up to ~13 MB the single launch wins; the 25.7 MB layers lose because the split path's
// second read of x already hits the 126 MB L2 inside the step, while the on-chip kernel
// serialises copy-in, conversion-bound reduction (F2F.F64.F32 runs at 16/clk/SM,
// tools/lab/convbench.cu) and write-out per CTA. 16-bit activations: off (0.1 no gain,
// 0.4 2% slower).
struct OnchipEnv {
  bool enabled = true;
  double max_frac4 = 0.40, max_frac2 = 0.0;  // fp32 / 16-bit activations
  int force_kc = 0, force_nch = 0;
  OnchipEnv() {
    enabled = getenv("CGBN_NO_ONCHIP") == nullptr;
    if (const char* e = getenv("CGBN_ONCHIP_MAX_FRAC")) max_frac4 = max_frac2 = atof(e);
    if (const char* e = getenv("CGBN_ONCHIP_FORCE")) sscanf(e, "%d,%d", &force_nch, &force_kc);
  }
};
const OnchipEnv& onchip_env() {
  static const OnchipEnv env;
  return env;
}

struct OnchipPlan {
  onchip::OGeom g;
  unsigned grid;
  size_t smem;
  int ve;
};

int device_attr(cudaDeviceAttr a, int fallback) {
  int dev = 0, v = 0;
  cudaGetDevice(&dev);
  if (cudaDeviceGetAttribute(&v, a, dev) != cudaSuccess || v <= 0) return fallback;
  return v;
}

// Resident CTAs per SM of `kernel` at `smem` dynamic bytes (cached).
std::map<std::tuple<const void*, int, size_t>, int> g_occ_smem;
template <class K>
int occupancy_smem(K kernel, size_t smem) {
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_tuple(reinterpret_cast<const void*>(kernel), dev, smem);
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    auto it = g_occ_smem.find(key);
    if (it != g_occ_smem.end()) return it->second;
  }
  smem_optin(kernel, (size_t)device_attr(cudaDevAttrMaxSharedMemoryPerBlockOptin, 232448));
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, onchip::kThreadsO, smem) !=
      cudaSuccess) {
    cudaGetLastError();
    occ = 0;
  }
  std::lock_guard<std::mutex> lk(g_cache_mu);
  g_occ_smem[key] = occ;
  return occ;
}

// Clusters of `kc` CTAs co-resident at `smem` dynamic bytes (cached).
std::map<std::tuple<const void*, int, int, size_t>, int> g_cluster_smem;
template <class K>
int64_t cluster_capacity_smem(K kernel, uint32_t kc, size_t smem) {
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_tuple(reinterpret_cast<const void*>(kernel), dev, (int)kc, smem);
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    auto it = g_cluster_smem.find(key);
    if (it != g_cluster_smem.end()) return it->second;
  }
  smem_optin(kernel, (size_t)device_attr(cudaDevAttrMaxSharedMemoryPerBlockOptin, 232448));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(kc * 64);
  cfg.blockDim = dim3(onchip::kThreadsO);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = kc;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kernel, &cfg) != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  std::lock_guard<std::mutex> lk(g_cache_mu);
  g_cluster_smem[key] = n;
  return n;
}

// ve == 16 / sizeof(T): the aligned instance; 1: odd planes (masked 16-byte covers)
template <class T, bool BWD, bool RELU>
auto onchip_kernel(int ve) {
  constexpr int ue = 16 / (int)sizeof(T);
  return ve == ue ? onchip::k_onchip<T, ue, BWD, RELU> : onchip::k_onchip<T, 1, BWD, RELU>;
}

// Choose (nch, KC): every CTA resident in one wave, the least bytes on the busiest SM.
template <class T, bool BWD, bool RELU>
bool onchip_plan_t(int64_t N, int64_t C, int64_t HW, OnchipPlan* p, bool capped) {
  constexpr int es = (int)sizeof(T);
  constexpr int nin = BWD ? 2 : 1;
  const OnchipEnv& env = onchip_env();
  // planes of whole 16-byte chunks (every run 16-byte aligned): the fast path; odd
  // planes read masked 16-byte covers, and a write chunk may span two channels (needs
  // HW >= 16 / sizeof(T))
  constexpr int ue = 16 / es;
  const int ve = HW % ue == 0 ? ue : 1;
  if (ve == 1 && HW < ue) return false;
  // the plan must not depend on RELU (the statistics-only launches use RELU = false for
  // the forward): every instance has the same registers, so plan on the RELU = false one
  auto kernel = onchip_kernel<T, BWD, false>(ve);
  const int64_t S = num_sms_cached();
  const int64_t smem_sm = device_attr(cudaDevAttrMaxSharedMemoryPerMultiprocessor, 233472);
  const int64_t smem_blk = device_attr(cudaDevAttrMaxSharedMemoryPerBlockOptin, 232448);
  const int64_t total = (int64_t)nin * N * C * HW * es;
  // capped: the automatic choice (the *_local / statistics entry points); uncapped: the
  // explicit *_fused entry points (any layer that fits in one resident wave)
  const double max_frac = !capped ? 1.0 : es == 4 ? env.max_frac4 : env.max_frac2;
  if ((double)total > max_frac * (double)(S * smem_sm)) return false;
  // a single image has no image split to spread over a cluster: with cold inputs the
  // split path measured slightly faster ([1,2048,7,7] fwd+bwd 11.9 vs 12.3 us,
  // tools/gpu/lat_sweep.sh, profiles/r2_knobs/lat_sweep/); the explicit *_fused entry
  // points still run it on chip
  if (capped && N == 1) return false;
  const size_t head = ((sizeof(onchip::Head) + 15) / 16) * 16;
  double best = 1e300;
  bool found = false;
  for (int64_t kc = 1; kc <= 8 && kc <= N; kc *= 2) {
    if (env.force_kc && kc != env.force_kc) continue;
    const int64_t nk = ceil_div(N, kc);
    if (nk > onchip::kMaxImg) continue;
    for (int64_t nch = 1; nch <= 1024; nch *= 2) {
      if (env.force_nch && nch != env.force_nch) continue;
      if (nch > 1 && (nch / 2) >= C) break;
      const int64_t run = nch * HW * es;
      const int64_t stride = (run + 15) / 16 * 16 + 16;
      const size_t smem = head + (onchip::chan_bytes<BWD>((uint32_t)nch) + 15) / 16 * 16 +
                          (size_t)(nk * nin * stride);
      if ((int64_t)smem > smem_blk) continue;
      const int64_t clusters = ceil_div(C, nch);
      const int64_t ctas = clusters * kc;
      const int cps = occupancy_smem(kernel, smem);
      if (cps < 1 || ctas > S * cps) continue;
      if (kc > 1 && clusters > cluster_capacity_smem(kernel, (uint32_t)kc, smem)) continue;
      // busiest SM: m = ceil(ctas / S) CTAs of nk * nin * run bytes. A lone CTA cannot
      // overlap its copy-in, reduction and write phases; m CTAs overlap each other's
      // (factor 1 + 1/m). A cluster level costs ~one barrier round trip (~0.5 us ~ 20 KB
      // at the per-SM HBM share).
      const double m = (double)ceil_div(ctas, S);
      const double score = m * (double)(nk * nin * run) * (1.0 + 1.0 / m) +
                           20e3 * (kc > 1 ? __builtin_ctzll(kc) : 0) + 64.0 * ctas;
      if (score < best) {
        best = score;
        found = true;
        onchip::OGeom& g = p->g;
        g.N = (uint32_t)N;
        g.C = (uint32_t)C;
        g.HW = (uint32_t)HW;
        g.nch = (uint32_t)nch;
        g.KC = (uint32_t)kc;
        g.run_stride = (uint32_t)stride;
        // aligned: the exact chunks of a run; else the slots of its 16-byte cover
        g.nq = (uint32_t)(ve == ue ? run / 16 : stride / 16);
        const int64_t wpc = nch >= onchip::kWarpsO ? 1 : onchip::kWarpsO / nch;
        g.wpc_log2 = (uint32_t)__builtin_ctzll(wpc);
        g.HWv = (uint32_t)(ve == ue ? HW / ue : (HW + ue - 1) / ue + 1);
        g.HWu = (uint32_t)(ve == ue ? HW / ue : 1);
        g.dhwv.init(g.HWv);
        g.dhw.init((uint32_t)HW);
        g.dhwu.init(g.HWu);
        g.dnq.init(g.nq);
        g.count = (double)(N * HW);
        p->grid = (unsigned)ctas;
        p->smem = smem;
        p->ve = ve;
      }
    }
  }
  return found;
}

// On-chip eligibility: NCHW planes of >= 4 elements, 16-byte aligned pointers and tensor
// size, the footprint within max_frac of the GPU's shared memory, one resident wave.
template <class T, bool BWD, bool RELU>
bool onchip_plan(int64_t N, int64_t C, int64_t HW, int layout, uintptr_t align,
                 OnchipPlan* p, bool capped = true) {
  if (!onchip_env().enabled || layout != CGBN_LAYOUT_NCHW || HW < 4) return false;
  if (align % 16 || ((uint64_t)N * C * HW * sizeof(T)) % 16) return false;
  if (validate_shape(N, C, HW, layout) != CGBN_OK) return false;
  if (!onchip_plan_t<T, BWD, RELU>(N, C, HW, p, capped)) return false;
  if (env().debug_plan)
    fprintf(stderr, "[cgbn] onchip %s N=%lld C=%lld HW=%lld -> nch=%u kc=%u grid=%u smem=%zu ve=%d\n",
            BWD ? "bwd" : "fwd", (long long)N, (long long)C, (long long)HW, p->g.nch, p->g.KC,
            p->grid, p->smem, p->ve);
  return true;
}

// Debug: per-CTA phase timestamps of the on-chip launches (cgbn_debug_onchip_trace).
unsigned long long* g_onchip_trace = nullptr;

template <class T, bool BWD, bool RELU>
int launch_onchip(const OnchipPlan& p, const onchip::Args& a0, cudaStream_t st) {
  auto kernel = onchip_kernel<T, BWD, RELU>(p.ve);
  smem_optin(kernel, (size_t)device_attr(cudaDevAttrMaxSharedMemoryPerBlockOptin, 232448));
  onchip::Args a = a0;
  a.trace = g_onchip_trace;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.grid);
  cfg.blockDim = dim3(onchip::kThreadsO);
  cfg.dynamicSmemBytes = p.smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  int na = 0;
  if (p.g.KC > 1) {
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = p.g.KC;
    at[na].val.clusterDim.y = 1;
    at[na].val.clusterDim.z = 1;
    ++na;
  }
  if (pdl_enabled()) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, p.g, a);
  if (e != cudaSuccess)
    return set_error(CGBN_ERR_CUDA, "on-chip launch failed: %s", cudaGetErrorString(e));
  return CGBN_OK;
}

// Try the on-chip pass; returns 1 if launched, 0 if not eligible, < 0 on error.
template <class T, bool BWD, bool RELU>
int try_onchip_t(int64_t N, int64_t C, int64_t HW, int layout, uintptr_t align,
                 const onchip::Args& a, cudaStream_t st, bool capped) {
  OnchipPlan p;
  if (!onchip_plan<T, BWD, RELU>(N, C, HW, layout, align, &p, capped)) return 0;
  const int rc = launch_onchip<T, BWD, RELU>(p, a, st);
  return rc == CGBN_OK ? 1 : -rc;
}

template <bool BWD>
int try_onchip(int act, bool relu, int64_t N, int64_t C, int64_t HW, int layout,
               uintptr_t align, const onchip::Args& a, cudaStream_t st, bool capped = true) {
  CGBN_ROUTED(act);
  return relu ? try_onchip_t<TuAct, BWD, true>(N, C, HW, layout, align, a, st, capped)
              : try_onchip_t<TuAct, BWD, false>(N, C, HW, layout, align, a, st, capped);
}

template <bool BWD>
bool onchip_supported(int act, bool relu, int64_t N, int64_t C, int64_t HW, int layout,
                      bool capped) {
  if (act != CGBN_TU_ACT) return false;
  OnchipPlan p;
  return relu ? onchip_plan<TuAct, BWD, true>(N, C, HW, layout, 0, &p, capped)
              : onchip_plan<TuAct, BWD, false>(N, C, HW, layout, 0, &p, capped);
}

#define CGBN_REQUIRE(cond, ...) \
  do { if (!(cond)) return set_error(CGBN_ERR_INVALID, __VA_ARGS__); } while (0)

#define CGBN_TRY(expr) \
  do { int rc_ = (expr); if (rc_) return rc_; } while (0)

int check_fwd_args(const void* x, const void* y, const float* gamma, const float* beta,
                   const double* saved, double eps, double momentum, const float* running_mean,
                   const float* running_var) {
  CGBN_REQUIRE(x && y && gamma && beta && saved, "forward: NULL pointer");
  CGBN_REQUIRE(eps > 0.0, "eps must be positive, got %g", eps);
  CGBN_REQUIRE(momentum >= 0.0 && momentum <= 1.0, "momentum must lie in [0, 1], got %g",
               momentum);
  CGBN_REQUIRE((running_mean == nullptr) == (running_var == nullptr),
               "running_mean and running_var must both be set or both be NULL");
  return CGBN_OK;
}

}  // namespace
