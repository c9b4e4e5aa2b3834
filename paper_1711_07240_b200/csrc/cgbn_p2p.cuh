// cgbn_p2p.cuh — one-shot peer-to-peer exchange of the per-rank statistics partial over
// NVLink / NVSwitch (SURVEY 8(e) backend 2; BASELINE north_star "latency-optimised
// one-shot P2P path measured against" NCCL). Included by cgbn.cu.
//
// Every rank of a BN group owns one region of device memory, shared with the group
// through CUDA IPC (cgbn_p2p_alloc / cgbn_p2p_open):
//
//   [ epoch counter (u64, local) | flags[G] (u64) | done | recv[2][G][max_len] (f64) ]
//
// (the `done` word serves the fused variant, where the statistics kernel's finishers push
// their channels directly and the finalize kernel waits: cgbn_*_p2p)
// One exchange = one single-CTA kernel per rank:
//   1. epoch = ++counter (device-side, so CUDA-graph replays advance it);
//   2. push: the rank writes its vector into recv[epoch & 1][rank] of every region
//      (peer stores over NVLink), fence.sc.sys;
//   3. publish: st.release.sys flags[rank] = epoch in every region;
//   4. wait: thread q spins on its own flags[q] >= epoch (ld.acquire.sys), with a
//      globaltimer timeout that sets CGBN_STATUS_EXCHANGE_TIMEOUT instead of hanging;
//   5. copy recv[epoch & 1][*] to a fixed output buffer, so the consumer kernel's
//      pointers stay valid across graph replays.
// Double buffering is sufficient: a peer can only write epoch e + 2 after every rank
// has published e + 1, i.e. after every rank's stream finished consuming epoch e.
// The fold over the G rows stays in the consumer kernels (ascending rank order), so
// the result is bitwise identical to the NCCL path.
//
// The same device routine runs in cgbn_p2p_emulate: a cooperative launch where CTA b
// plays rank b on regions of one GPU (all CTAs co-resident, as for a grid barrier),
// which validates the protocol on a single GPU without separately launched kernels
// waiting on one another.

#pragma once

namespace {
namespace p2p {

constexpr int kThreadsP2P = 256;
constexpr int kMaxPeers = CGBN_MAX_GROUP;

struct Peers {
  char* base[kMaxPeers];  // region of every rank of the group (own at [rank])
};

// (region layout, flags and the acquire / release helpers: cgbn_common.cuh)

// One rank's exchange, executed by one CTA (blockDim.x threads, >= G).
__device__ void exchange_rank(const double* __restrict__ vec, int64_t n, int rank, int G,
                              const Peers& peers, int64_t max_len, double* __restrict__ out,
                              unsigned* status, uint64_t timeout_ns) {
  __shared__ unsigned long long s_epoch;
  __shared__ unsigned s_missing;  // bit q: rank q did not publish in time
  char* mine = peers.base[rank];
  if (threadIdx.x == 0) {
    unsigned long long* ctr = reinterpret_cast<unsigned long long*>(mine);
    s_epoch = *ctr + 1;
    *ctr = s_epoch;
    s_missing = 0u;
  }
  __syncthreads();
  const unsigned long long e = s_epoch;
  const int par = (int)(e & 1ull);
  // 2. push my vector to every rank (own region included)
  for (int q = 0; q < G; ++q) {
    double* dst = recv_ptr(peers.base[q], G, max_len, par, rank);
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) dst[i] = vec[i];
  }
  __threadfence_system();
  __syncthreads();
  // 3. publish (thread q signals rank q)
  if ((int)threadIdx.x < G) st_release_sys(flag_ptr(peers.base[threadIdx.x], rank), e);
  // 4. wait for every rank's epoch-e data in my region
  if ((int)threadIdx.x < G) {
    const unsigned long long* f = flag_ptr(mine, threadIdx.x);
    const uint64_t t0 = now_ns();
    while (ld_acquire_sys(f) < e) {
      if (now_ns() - t0 > timeout_ns) {
        if (status) atomicOr(status, CGBN_STATUS_EXCHANGE_TIMEOUT);
        atomicOr(&s_missing, 1u << threadIdx.x);
        break;
      }
    }
  }
  __syncthreads();
  __threadfence_system();
  // 5. rows in rank order into the fixed output buffer; a missing rank's row is NaN (its
  // slot still holds an older exchange), so nothing downstream folds stale statistics
  const unsigned missing = s_missing;
  for (int q = 0; q < G; ++q) {
    const double* src = recv_ptr(mine, G, max_len, par, q);
    const bool miss = (missing >> q) & 1u;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x)
      out[(size_t)q * n + i] = miss ? __longlong_as_double(0x7ff8000000000000ll) : src[i];
  }
}

__global__ void __launch_bounds__(kThreadsP2P)
k_p2p_exchange(const double* vec, int64_t n, int rank, int G, Peers peers, int64_t max_len,
               double* out, unsigned* status, uint64_t timeout_ns) {
  pdl_wait();  // the partial comes from the previous kernel
  exchange_rank(vec, n, rank, G, peers, max_len, out, status, timeout_ns);
  pdl_trigger();
}

// Single-GPU protocol check: CTA b is rank b (cooperative launch: all co-resident).
// `skip` >= 0 makes that rank sit the exchange out (timeout path).
__global__ void __launch_bounds__(kThreadsP2P)
k_p2p_emulate(const double* vecs, int64_t n, int G, Peers peers, int64_t max_len, double* outs,
              unsigned* status, uint64_t timeout_ns, int skip) {
  const int b = blockIdx.x;
  if (b == skip) return;
  exchange_rank(vecs + (size_t)b * n, n, b, G, peers, max_len, outs + (size_t)b * G * n,
                status, timeout_ns);
}

}  // namespace p2p
}  // namespace
