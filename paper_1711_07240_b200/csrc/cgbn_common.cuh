// cgbn_common.cuh — errors, reduction geometry and the unit cursor, typed vector I/O, load rounds
// Part of the single translation unit cgbn.cu (included there, in order).

#pragma once

// The thread-local message behind cgbn_last_error() (defined once, in unit 0 of cgbn.cu).
int cgbn_internal_set_error(int code, const char* msg);

namespace {

// ----------------------------------------------------------------------------------
// Errors

static int set_error(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  return cgbn_internal_set_error(code, buf);
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess)
    return set_error(CGBN_ERR_CUDA, "%s: CUDA launch failed: %s", what, cudaGetErrorString(e));
  return CGBN_OK;
}

// ----------------------------------------------------------------------------------
// Geometry

// Unsigned 32-bit division by a runtime-constant divisor, valid for every n < 2^32
// (Hacker's Delight round-up method): t = umulhi(n, m), q = (t + ((n - t) >> s1)) >> s2
// with l = ceil(log2 d), m = floor(2^32 (2^l - d) / d) + 1, s1 = min(l, 1), s2 = l - s1.
struct FastDiv {
  uint32_t m, s1, s2;
  void init(uint32_t d) {
    uint32_t l = 0;
    while ((1ull << l) < d) ++l;
    m = (uint32_t)(((1ull << 32) * ((1ull << l) - d)) / d + 1);
    s1 = l < 1 ? l : 1;
    s2 = l - s1;
  }
  __device__ __forceinline__ uint32_t div(uint32_t n) const {
    const uint32_t t = __umulhi(n, m);
    return (t + ((n - t) >> s1)) >> s2;
  }
};

// Reduction-kernel geometry. Element offset of vector unit j of channel c:
// (c*HWv + j + (j / HWv) * gap) * VEC with gap = (C-1)*HWv. NCHW: HWv = HW/VEC.
// NHWC and 2-D (N, C): HWv = 1, VEC = 1.
// VM (vector mode) 1, 2, 4: exact vectors of VM floats (HW % VM == 0); VM 5 = "masked
// float4": planes whose length is not a multiple of 4 (ResNet 7x7, FPN 25x42 / 13x21) are
// read as the aligned float4 cover of each plane (ceil(HW/4) + 1 units per plane) with a
// per-element mask, so odd planes also stream with 128-bit loads.
struct Geom {
  uint32_t C;
  uint32_t Lv;        // vector units per channel stream (N*HWv)
  uint32_t HWv;       // vector units per plane
  uint32_t grid;      // CTAs of this launch
  uint32_t tpc_log2;  // team kernels: log2(threads per channel)
  uint32_t HW;        // floats per plane (1 for NHWC / 2-D)
  uint64_t T;         // C * Lv
  uint64_t gap;       // (C-1)*HWv
  FastDiv dhw;        // division by HWv
  double count;       // elements per channel on this rank (N*HW)
};

// Vector modes (elements per load unit): 1, 2, 4, 8 exact; 5 = masked 4-element cover
// (fp32), 9 = masked 8-element cover (bf16 / fp16). A unit is at most 16 bytes.
constexpr int vec_of(int vm) { return vm == 5 ? 4 : vm == 9 ? 8 : vm; }
constexpr bool masked_vm(int vm) { return vm == 5 || vm == 9; }

// Unit cursor: the position of one thread in a channel stream, advanced by a fixed
// stride without a division per unit. P = (n*C + c)*HWv is the vector-unit index of the
// start of plane (n, c), o the unit within the plane, ps = (n*C + c)*HW the plane start
// in floats (masked mode). All fit in 32 bits (N*C*HW < 2^32). tools/flatlab.cu measured
// the per-unit FastDiv + 64-bit multiply addressing at 1.2-2 us per launch on ResNet
// mid shapes.
struct Cursor {
  uint32_t P, o, ps;
};

struct Step {
  uint32_t q, r;  // stride = q*HWv + r
};

__device__ __forceinline__ Cursor cursor_at(const Geom& g, uint32_t c, uint32_t j) {
  const uint32_t n = g.dhw.div(j);
  const uint32_t nc = n * g.C + c;
  return Cursor{nc * g.HWv, j - n * g.HWv, nc * g.HW};
}

__device__ __forceinline__ Step step_of(const Geom& g, uint32_t stride) {
  const uint32_t q = g.dhw.div(stride);
  return Step{q, stride - q * g.HWv};
}

__device__ __forceinline__ void advance(const Geom& g, Cursor& k, const Step& s) {
  const uint32_t CHWv = g.C * g.HWv, CHW = g.C * g.HW;
  k.o += s.r;
  k.P += s.q * CHWv;
  k.ps += s.q * CHW;
  if (k.o >= g.HWv) {
    k.o -= g.HWv;
    k.P += CHWv;
    k.ps += CHW;
  }
}

// Address (in floats) and element mask of the unit under the cursor.
template <int VM>
__device__ __forceinline__ uint32_t unit_addr(const Geom& g, const Cursor& k, uint32_t& mask) {
  constexpr uint32_t V = vec_of(VM);
  if constexpr (!masked_vm(VM)) {
    mask = (1u << V) - 1u;
    return (k.P + k.o) * V;
  } else {
    const uint32_t base = (k.ps & ~(V - 1u)) + V * k.o;
    const int lo = (int)(k.ps - base);            // plane start relative to the unit
    const int hi = lo + (int)g.HW;                // plane end relative to the unit
    mask = 0u;
#pragma unroll
    for (int e = 0; e < (int)V; ++e) mask |= (e >= lo && e < hi) ? (1u << e) : 0u;
    return base;
  }
}

// flat: CTA b owns stream units [cta_begin(b), cta_begin(b+1)).
__device__ __forceinline__ uint64_t cta_begin(const Geom& g, uint32_t b) {
  return (uint64_t)b * g.T / g.grid;
}
// The CTA whose slice contains unit u: the largest b with cta_begin(b) <= u.
__device__ __forceinline__ uint32_t cta_of(const Geom& g, uint64_t u) {
  return (uint32_t)(((u + 1) * (uint64_t)g.grid - 1) / g.T);
}

struct Seg {
  uint32_t c, j0, j1;
};

template <class F>
__device__ __forceinline__ void for_each_segment(const Geom& g, F&& f) {
  const uint64_t u_end = cta_begin(g, blockIdx.x + 1);
  for (uint64_t u = cta_begin(g, blockIdx.x); u < u_end;) {
    const uint32_t c = (uint32_t)(u / g.Lv);
    const uint64_t cbase = (uint64_t)c * g.Lv;
    const uint64_t s_end = min(u_end, cbase + g.Lv);
    f(Seg{c, (uint32_t)(u - cbase), (uint32_t)(s_end - cbase)});
    u = s_end;
  }
}

struct Parts {
  const double* p[CGBN_MAX_GROUP];
  int G;
};

}  // namespace

// ----------------------------------------------------------------------------------
// One-shot P2P exchange regions (cgbn_p2p.cuh; fused into the reductions' finishers by
// the *_p2p entry points). Every rank of a BN group owns one region, shared with the group
// through CUDA IPC:
//   [ epoch counter (u64) | flags[G] (u64) | done (u32, padded) | recv[2][G][max_len] (f64) ]
// `done` counts the channel finishers of a fused reduction; the last one publishes.
namespace {
namespace p2p {

__host__ __device__ inline size_t flags_off() { return 8; }
__host__ __device__ inline size_t done_off(int G) { return 8 + (size_t)G * 8; }
__host__ __device__ inline size_t recv_off(int G) { return (done_off(G) + 8 + 15) / 16 * 16; }
__host__ __device__ inline size_t region_bytes(int G, int64_t max_len) {
  return recv_off(G) + 2 * (size_t)G * (size_t)max_len * sizeof(double);
}

__device__ __forceinline__ unsigned long long* flag_ptr(char* region, int q) {
  return reinterpret_cast<unsigned long long*>(region + flags_off()) + q;
}
__device__ __forceinline__ double* recv_ptr(char* region, int G, int64_t max_len, int parity,
                                            int q) {
  return reinterpret_cast<double*>(region + recv_off(G)) +
         ((size_t)parity * G + q) * (size_t)max_len;
}

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t now_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// The producer side of a fused exchange: this rank's row of every region, epoch parity
// from the own region's counter (read by every finisher before the last one advances it).
// At most kMaxPush ranks (one NVSwitch box): the pointers stay a small, statically
// indexed part of every reduction Op's kernel parameters.
constexpr int kMaxPush = 8;
struct Push {
  char* base[kMaxPush];  // region of every rank of the group (own at [rank])
  int rank, G;           // G == 0: no push (the finisher writes `out`)
  int64_t max_len;
  unsigned nfinish;      // finisher calls per launch (one per channel)
};

__device__ __forceinline__ char* push_own(const Push& P) {
  char* own = nullptr;
#pragma unroll
  for (int q = 0; q < kMaxPush; ++q)
    if (q == P.rank) own = P.base[q];
  return own;
}
__device__ __forceinline__ unsigned long long push_epoch(const Push& P) {
  return *reinterpret_cast<volatile unsigned long long*>(push_own(P)) + 1ull;
}

// After a finisher wrote its channel into every region: fence, count, and the last
// finisher advances the epoch and publishes this rank's flag in every region.
__device__ __forceinline__ void push_done(const Push& P, unsigned long long e) {
  __threadfence_system();
  char* own = push_own(P);
  unsigned* done = reinterpret_cast<unsigned*>(own + done_off(P.G));
  if (atomicAdd(done, 1u) == P.nfinish - 1) {
    *done = 0u;
    *reinterpret_cast<volatile unsigned long long*>(own) = e;
    __threadfence_system();
#pragma unroll
    for (int q = 0; q < kMaxPush; ++q)
      if (q < P.G) st_release_sys(flag_ptr(P.base[q], P.rank), e);
  }
}

// The consumer side: wait for every rank's flag of the current epoch (own counter), with
// a globaltimer timeout that sets CGBN_STATUS_EXCHANGE_TIMEOUT instead of hanging.
struct Pull {
  char* own;
  int G;
  int64_t max_len;
  unsigned* status;
  uint64_t timeout_ns;
};

// Called by every thread of a block; returns the epoch. Threads q < G spin on flag q.
// `timed_out` tells every thread that some rank never published: its rows still hold an
// older exchange, so the caller must not use them (collectives.py:138-144 raises before
// any state changes).
__device__ __forceinline__ unsigned long long pull_wait(const Pull& P, bool& timed_out) {
  __shared__ int s_timeout;
  if (threadIdx.x == 0) s_timeout = 0;
  __syncthreads();
  const unsigned long long e = *reinterpret_cast<volatile unsigned long long*>(P.own);
  if ((int)threadIdx.x < P.G) {
    const unsigned long long* f = flag_ptr(P.own, threadIdx.x);
    const uint64_t t0 = now_ns();
    while (ld_acquire_sys(f) < e) {
      if (now_ns() - t0 > P.timeout_ns) {
        if (P.status) atomicOr(P.status, CGBN_STATUS_EXCHANGE_TIMEOUT);
        s_timeout = 1;
        break;
      }
    }
  }
  __syncthreads();
  __threadfence_system();
  timed_out = s_timeout != 0;
  return e;
}

}  // namespace p2p
}  // namespace

namespace {

// ----------------------------------------------------------------------------------
// Vector load / store of activation elements (fp32, bf16 or fp16 storage; every kernel
// computes in fp64 and rounds once on output).

template <class T>
__device__ __forceinline__ float h2f(unsigned short h);
template <>
__device__ __forceinline__ float h2f<__nv_bfloat16>(unsigned short h) {
  return __bfloat162float(__ushort_as_bfloat16(h));
}
template <>
__device__ __forceinline__ float h2f<__half>(unsigned short h) {
  return __half2float(__ushort_as_half(h));
}

// one element, as float
template <class T>
__device__ __forceinline__ float ld1(const T* __restrict__ p) {
  if constexpr (sizeof(T) == 4) return __ldg(reinterpret_cast<const float*>(p));
  else return h2f<T>(__ldg(reinterpret_cast<const unsigned short*>(p)));
}

// fp64 -> storage, rounded once
template <class T>
__device__ __forceinline__ uint32_t rnd(double v) {
  if constexpr (sizeof(T) == 4) return __float_as_uint((float)v);
  else if constexpr (std::is_same<T, __nv_bfloat16>::value)
    return __bfloat16_as_ushort(__double2bfloat16(v));
  else return __half_as_ushort(__double2half(v));
}

template <class T>
__device__ __forceinline__ void st1(T* p, double v) {
  if constexpr (sizeof(T) == 4) *reinterpret_cast<float*>(p) = (float)v;
  else *reinterpret_cast<unsigned short*>(p) = (unsigned short)rnd<T>(v);
}

// V elements of T held as raw 32-bit words (the registers of one vector load).
template <class T, int V>
struct Vec {
  static constexpr int kBytes = V * (int)sizeof(T);
  static constexpr int kWords = kBytes >= 4 ? kBytes / 4 : 1;
  uint32_t w[kWords];
  __device__ __forceinline__ void load(const T* __restrict__ p) {
    if constexpr (kBytes == 16) {
      const uint4 t = __ldg(reinterpret_cast<const uint4*>(p));
      w[0] = t.x; w[1] = t.y; w[2] = t.z; w[3] = t.w;
    } else if constexpr (kBytes == 8) {
      const uint2 t = __ldg(reinterpret_cast<const uint2*>(p));
      w[0] = t.x; w[1] = t.y;
    } else if constexpr (kBytes == 4) {
      w[0] = __ldg(reinterpret_cast<const unsigned*>(p));
    } else {
      w[0] = __ldg(reinterpret_cast<const unsigned short*>(p));
    }
  }
  __device__ __forceinline__ float get(int k) const {
    if constexpr (sizeof(T) == 4) return __uint_as_float(w[k]);
    else return h2f<T>((unsigned short)(w[k >> 1] >> (16 * (k & 1))));
  }
};

// Round V fp64 values to T and store them as one vector.
template <class T, int V>
__device__ __forceinline__ void stv(T* __restrict__ p, const double (&t)[V]) {
  if constexpr (sizeof(T) == 4) {
    if constexpr (V == 4) {
      *reinterpret_cast<float4*>(p) = make_float4((float)t[0], (float)t[1], (float)t[2], (float)t[3]);
    } else {
#pragma unroll
      for (int k = 0; k < V; ++k) reinterpret_cast<float*>(p)[k] = (float)t[k];
    }
  } else {
    static_assert(V % 2 == 0, "16-bit stores pack pairs");
    uint32_t w[V / 2];
#pragma unroll
    for (int k = 0; k < V / 2; ++k) w[k] = rnd<T>(t[2 * k]) | (rnd<T>(t[2 * k + 1]) << 16);
    if constexpr (V == 8) *reinterpret_cast<uint4*>(p) = make_uint4(w[0], w[1], w[2], w[3]);
    else if constexpr (V == 4) *reinterpret_cast<uint2*>(p) = make_uint2(w[0], w[1]);
    else *reinterpret_cast<uint32_t*>(p) = w[0];
  }
}

// Round V fp32 values to the 16-bit T (pairs packed, one F2FP each) and store them as one
// vector (the fp32 elementwise path of 16-bit activations).
template <class T, int V>
__device__ __forceinline__ void stvf(T* __restrict__ p, const float (&t)[V]) {
  static_assert(sizeof(T) == 2 && V % 2 == 0, "16-bit pairs");
  uint32_t w[V / 2];
#pragma unroll
  for (int k = 0; k < V / 2; ++k) {
    if constexpr (std::is_same<T, __nv_bfloat16>::value) {
      const __nv_bfloat162 b = __floats2bfloat162_rn(t[2 * k], t[2 * k + 1]);
      w[k] = *reinterpret_cast<const uint32_t*>(&b);
    } else {
      const __half2 b = __floats2half2_rn(t[2 * k], t[2 * k + 1]);
      w[k] = *reinterpret_cast<const uint32_t*>(&b);
    }
  }
  if constexpr (V == 8) *reinterpret_cast<uint4*>(p) = make_uint4(w[0], w[1], w[2], w[3]);
  else if constexpr (V == 4) *reinterpret_cast<uint2*>(p) = make_uint2(w[0], w[1]);
  else *reinterpret_cast<uint32_t*>(p) = w[0];
}

// Loads in flight per thread per round: 64 B for one input stream, 32 B total for two
// (NIN = number of input streams).
// Round 2, measured on the ResNet-50 steps (profiles/r2_red_ab/): 8 / 4 (round 1) ->
// 4 / 2 kept the fp32 step (2.095 -> 2.092 ms) without the 16-124 B spills of 60 fp32
// reduction instantiations at the 64-register cap and sped up bf16 (1.525 -> 1.468 ms);
// 4 / 1 then gained the backward reduction another 3-5% (fp32 2.091 -> 2.077 ms, bf16
// 1.468 -> 1.449 ms); 2 / 1 lost on the statistics.
#ifndef CGBN_RED_U1
#define CGBN_RED_U1 4  // loads in flight per thread per round, one input stream
#endif
#ifndef CGBN_RED_U2
#define CGBN_RED_U2 1  // units per round with two input streams (dy, x)
#endif
#ifndef CGBN_CT_MINB
#define CGBN_CT_MINB 4  // k_reduce_ct CTAs per SM (register bound)
#endif
template <int VM, int NIN = 1>
constexpr int unroll_for() { return (NIN == 1 || VM == 1) ? CGBN_RED_U1 : CGBN_RED_U2; }

// Visit units j = start, start+stride, ... < end of channel c in rounds of U: the U
// (predicated) loads of a round are issued before any of them is used.
template <int U, class Op, class Body>
__device__ __forceinline__ void strided_rounds(const Geom& g, uint32_t c, uint32_t start,
                                               uint32_t end, uint32_t stride, const Op& op,
                                               Body&& body) {
  if (start >= end) return;
  Cursor k = cursor_at(g, c, start);
  const Step s = step_of(g, stride);
  for (uint32_t i = start; i < end; i += U * stride) {
    typename Op::Regs r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t j = i + u * stride;
      if (j < end) op.load(g, k, r[u]);
      advance(g, k, s);  // after U steps: the next round's first unit
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t j = i + u * stride;
      if (j < end) body(u, j, r[u]);
    }
  }
}

}  // namespace
