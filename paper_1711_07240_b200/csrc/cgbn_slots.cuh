// cgbn_slots.cuh — the producer's per-CTA statistics slots and their merge, shared by
// the conv (cgbn_conv.cu: k_conv_fold -> rank partial) and the BN finalize
// (cgbn.cu: k_finalize_slots -> coefficients directly, single-rank groups).
//
// Slot table (the conv's statistics workspace): a 32-byte header
// {nslots, mtiles, grid, Cout} written by the conv kernel, then Slot[nslots][Cout].
// Slot s of channel c exists when CTA (s / 2) * mtiles + c / 128 ran.
#pragma once

namespace cgbn_slots {

struct Slot {
  double n, mean, M2;
};

struct Header {
  int nslots, mtiles, grid, cout;
  int pad[4];
};
static_assert(sizeof(Header) == 32, "slot table header is 32 bytes");

constexpr int kFoldPerWarp = 10;  // slots per channel <= 2 * 148 CTAs <= 32 warps x 10

__host__ __device__ inline const Slot* table(const void* ws) {
  return reinterpret_cast<const Slot*>(static_cast<const char*>(ws) + sizeof(Header));
}

// Merge of channel c's slots by a 32 x 32 block (lane = channel, warp w takes slots w,
// w + 32, ...) against one shift K0 = the first non-empty slot's mean: A = sum n_k (mean_k - K0), B = sum
// M2_k + n_k (mean_k - K0)^2 (additions only), the 32 warp sums added in warp order by
// warp 0, which gets (n, mean, M2); other warps' results are meaningless. Fixed order:
// bitwise reproducible.
__device__ __forceinline__ void merge(const Slot* __restrict__ slots, int Cout, int mtiles,
                                      int grid, int nslots, int c, double (&sn)[32][32],
                                      double (&sa)[32][32], double (&sb)[32][32], double& n_out,
                                      double& mean_out, double& M2_out) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int mt = c / 128;
  double n = 0.0, A = 0.0, B = 0.0, K0 = 0.0;
  if (c < Cout) {
    Slot p[kFoldPerWarp];
    // the shift: the first non-empty slot's mean (a CTA that only ran non-final split-K
    // ranges leaves n = 0 slots)
    for (int s = 0; s < nslots; ++s) {
      if ((s >> 1) * mtiles + mt >= grid) continue;
      const Slot q = slots[(size_t)s * Cout + c];
      if (q.n > 0.0) {
        K0 = q.mean;
        break;
      }
    }
    // two halves of kFoldPerWarp / 2 loads in flight (all of them at once spilled at the
    // 1024-thread block's 64-register cap); the adds keep the u order
    constexpr int kHalf = kFoldPerWarp / 2;
#pragma unroll
    for (int h = 0; h < kFoldPerWarp; h += kHalf) {
#pragma unroll
      for (int u = h; u < h + kHalf; ++u) {
        const int s = w + 32 * u;
        const bool ok = s < nslots && (s >> 1) * mtiles + mt < grid;
        p[u] = ok ? slots[(size_t)s * Cout + c] : Slot{0.0, 0.0, 0.0};
      }
#pragma unroll
      for (int u = h; u < h + kHalf; ++u) {
        if (p[u].n == 0.0) continue;
        const double d = p[u].mean - K0;
        n += p[u].n;
        A = fma(p[u].n, d, A);
        B += fma(p[u].n * d, d, p[u].M2);
      }
    }
  }
  sn[w][lane] = n;
  sa[w][lane] = A;
  sb[w][lane] = B;
  __syncthreads();
  if (w == 0 && c < Cout) {
    for (int r = 1; r < 32; ++r) {
      n += sn[r][lane];
      A += sa[r][lane];
      B += sb[r][lane];
    }
  }
  n_out = n;
  mean_out = K0 + A / n;
  M2_out = B - A * A / n;
}

}  // namespace cgbn_slots
