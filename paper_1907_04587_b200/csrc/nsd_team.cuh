// Execution teams for the Newton-step engine.
//
// The whole per-timestep solve (nsd_engine.cuh) is written once against a
// "team": a set of threads that cooperatively owns one scene. A team exposes
// rank/size for strided work loops, a barrier, and a deterministic all-reduce
// (fixed summation order; every member receives the identical bits, so all
// data-dependent branches — PCR exits, breakdown, abort — are team-uniform).
//
//   WarpTeam  — one warp per environment (batched RL path, tiny scenes):
//               barrier = __syncwarp, reductions = shuffle trees.
//   BlockTeam — one CTA per scene/environment: barrier = __syncthreads,
//               reductions through double-buffered shared memory.
//   GridTeam  — a cooperative persistent grid per large scene (FEM configs):
//               barrier = grid-wide sync, reductions through per-CTA partials
//               in global memory summed in CTA order.
#pragma once

#include <cooperative_groups.h>

namespace nsd {

constexpr int kRedMax = 8;  // max values per fused reduction

__device__ __forceinline__ double warp_sum_down(double v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
  return v;
}
__device__ __forceinline__ double warp_max_down(double v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v = fmax(v, __shfl_down_sync(0xffffffffu, v, off));
  return v;
}

struct WarpTeam {
  int lane;
  __device__ explicit WarpTeam(int l) : lane(l) {}
  __device__ __forceinline__ int rank() const { return lane; }
  __device__ __forceinline__ int size() const { return 32; }
  __device__ __forceinline__ void sync() const { __syncwarp(); }
  // sums s[0..NS), maxima m[0..NM); results broadcast from lane 0.
  template <int NS, int NM>
  __device__ __forceinline__ void reduce(double (&s)[NS], double (&m)[NM]) {
    __syncwarp();
#pragma unroll
    for (int k = 0; k < NS; ++k) s[k] = __shfl_sync(0xffffffffu, warp_sum_down(s[k]), 0);
#pragma unroll
    for (int k = 0; k < NM; ++k) m[k] = __shfl_sync(0xffffffffu, warp_max_down(m[k]), 0);
  }
  template <int NS> __device__ __forceinline__ void reduce_sum(double (&s)[NS]) {
    __syncwarp();
#pragma unroll
    for (int k = 0; k < NS; ++k) s[k] = __shfl_sync(0xffffffffu, warp_sum_down(s[k]), 0);
  }
};

// TPE consecutive lanes of a warp per environment (TPE in {4, 8, 16, 32}).
// Shuffles and barriers use the team's own lane mask, so the teams sharing a
// warp may take different data-dependent paths (PCR exits, aborts) safely.
template <int TPE> struct SubWarpTeam {
  static_assert(TPE == 4 || TPE == 8 || TPE == 16 || TPE == 32, "TPE");
  static constexpr int kSize = TPE;
  int lane;       // rank within the team
  unsigned mask;  // the team's lanes
  __device__ explicit SubWarpTeam(int warp_lane)
      : lane(warp_lane & (TPE - 1)),
        mask(TPE == 32 ? 0xffffffffu : (((1u << TPE) - 1u) << (warp_lane & ~(TPE - 1)))) {}
  __device__ __forceinline__ int rank() const { return lane; }
  __device__ __forceinline__ int size() const { return TPE; }
  __device__ __forceinline__ void sync() const { __syncwarp(mask); }
  template <int NS, int NM>
  __device__ __forceinline__ void reduce(double (&s)[NS], double (&m)[NM]) {
    __syncwarp(mask);
#pragma unroll
    for (int k = 0; k < NS; ++k) {
      double v = s[k];
#pragma unroll
      for (int off = TPE / 2; off > 0; off >>= 1) v += __shfl_down_sync(mask, v, off, TPE);
      s[k] = __shfl_sync(mask, v, 0, TPE);
    }
#pragma unroll
    for (int k = 0; k < NM; ++k) {
      double v = m[k];
#pragma unroll
      for (int off = TPE / 2; off > 0; off >>= 1) v = fmax(v, __shfl_down_sync(mask, v, off, TPE));
      m[k] = __shfl_sync(mask, v, 0, TPE);
    }
  }
  template <int NS> __device__ __forceinline__ void reduce_sum(double (&s)[NS]) {
    __syncwarp(mask);
    double v[NS];
#pragma unroll
    for (int k = 0; k < NS; ++k) v[k] = s[k];
#pragma unroll
    for (int off = TPE / 2; off > 0; off >>= 1)
#pragma unroll
      for (int k = 0; k < NS; ++k) v[k] += __shfl_down_sync(mask, v[k], off, TPE);
#pragma unroll
    for (int k = 0; k < NS; ++k) s[k] = __shfl_sync(mask, v[k], 0, TPE);
  }
};

struct BlockTeam {
  double* red;  // shared: 2 * (33 * kRedMax) doubles
  int parity;
  __device__ explicit BlockTeam(double* smem_red) : red(smem_red), parity(0) {}
  __device__ __forceinline__ int rank() const { return threadIdx.x; }
  __device__ __forceinline__ int size() const { return blockDim.x; }
  __device__ __forceinline__ void sync() const { __syncthreads(); }
  template <int NS> __device__ __forceinline__ void reduce_sum(double (&s)[NS]) {
    double m[1] = {0.0};
    reduce(s, m);
  }
  template <int NS, int NM>
  __device__ __forceinline__ void reduce(double (&s)[NS], double (&m)[NM]) {
    constexpr int K = NS + NM;
    static_assert(K <= kRedMax, "too many values in one reduction");
    double* buf = red + parity * (33 * kRedMax);
    parity ^= 1;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int k = 0; k < NS; ++k) {
      const double v = warp_sum_down(s[k]);
      if (lane == 0) buf[warp * kRedMax + k] = v;
    }
#pragma unroll
    for (int k = 0; k < NM; ++k) {
      const double v = warp_max_down(m[k]);
      if (lane == 0) buf[warp * kRedMax + NS + k] = v;
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
      for (int k = 0; k < NS; ++k) {
        const double v = warp_sum_down(lane < nw ? buf[lane * kRedMax + k] : 0.0);
        if (lane == 0) buf[32 * kRedMax + k] = v;
      }
#pragma unroll
      for (int k = 0; k < NM; ++k) {
        const double v = warp_max_down(lane < nw ? buf[lane * kRedMax + NS + k] : -__builtin_huge_val());
        if (lane == 0) buf[32 * kRedMax + NS + k] = v;
      }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < NS; ++k) s[k] = buf[32 * kRedMax + k];
#pragma unroll
    for (int k = 0; k < NM; ++k) m[k] = buf[32 * kRedMax + NS + k];
  }
};

// Grid team: one cooperative launch, one CTA per SM. Barrier and all-reduce are
// "last CTA reduces": each CTA publishes its partials and arrives on a global
// counter; the last to arrive sums the partials in CTA order (deterministic,
// bit-identical for every member), publishes the totals and bumps a generation
// flag that the other CTAs spin on. One barrier-equivalent per reduction, and
// only one CTA reads the partials (measured: the previous scheme — a CG grid sync
// after which every CTA's warp 0 re-read all partials, value by value, from the
// same L2 lines — held ~48% of the C2 kernel's stall samples).
// Global scratch (gpart): [2 x nb x kRedMax partials][2 x kRedMax totals][count, gen];
// count and gen are zeroed before every launch.
struct GridTeam {
  double* red;    // shared: 2 * (33 * kRedMax)
  double* gpart;  // global partials
  double* gres;   // global totals
  unsigned* bar;  // [0] arrival count, [1] generation
  int parity;
  unsigned epoch;
  __device__ GridTeam(double* smem_red, double* global_part)
      : red(smem_red), gpart(global_part), gres(global_part + 2 * gridDim.x * kRedMax),
        bar(reinterpret_cast<unsigned*>(global_part + 2 * gridDim.x * kRedMax + 2 * kRedMax)), parity(0), epoch(0) {}
  __device__ __forceinline__ int rank() const { return blockIdx.x * blockDim.x + threadIdx.x; }
  __device__ __forceinline__ int size() const { return gridDim.x * blockDim.x; }

  // Arrive; returns true (block-uniform) in the last CTA to arrive. The arrival
  // count only grows within a launch (zeroed by the host before each launch): a
  // CTA reaches barrier n + 1 only after every CTA arrived at barrier n, so the
  // last arriver of barrier n sees a count of n * gridDim.x. The acq_rel atomic
  // publishes thread 0's writes (the CTA partials; other threads' writes are
  // ordered before it by the __syncthreads) and, in the last arriver, acquires
  // every earlier arriver's — one L2 round trip, no separate fence.
  __device__ __forceinline__ bool arrive(int* last_flag) {
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned prev;
      asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(bar) : "memory");
      *last_flag = (prev + 1u) % gridDim.x == 0u;
    }
    __syncthreads();
    return *last_flag != 0;
  }
  // Last CTA: release the waiting CTAs (its writes, ordered before thread 0 by
  // __syncthreads, are published by the release store); others: wait.
  __device__ __forceinline__ void release_or_wait(bool last) {
    ++epoch;
    if (threadIdx.x == 0) {
      if (last) {
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(bar + 1), "r"(epoch) : "memory");
      } else {
        unsigned g;
        do {  // acquire load: no atomic traffic on the hot word while waiting
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(bar + 1) : "memory");
        } while (g != epoch);
      }
    }
    __syncthreads();
  }

  __device__ __forceinline__ void sync() {
    __shared__ int last_flag;
    const bool last = arrive(&last_flag);
    release_or_wait(last);
  }
  template <int NS> __device__ __forceinline__ void reduce_sum(double (&s)[NS]) {
    double m[1] = {0.0};
    reduce(s, m);
  }
  template <int NS, int NM>
  __device__ __forceinline__ void reduce(double (&s)[NS], double (&m)[NM]) {
    constexpr int K = NS + NM;
    static_assert(K <= kRedMax, "too many values in one reduction");
    __shared__ int last_flag;
    double* buf = red + parity * (33 * kRedMax);
    double* gp = gpart + parity * (gridDim.x * kRedMax);
    double* gr = gres + parity * kRedMax;
    parity ^= 1;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int k = 0; k < NS; ++k) {
      const double v = warp_sum_down(s[k]);
      if (lane == 0) buf[warp * kRedMax + k] = v;
    }
#pragma unroll
    for (int k = 0; k < NM; ++k) {
      const double v = warp_max_down(m[k]);
      if (lane == 0) buf[warp * kRedMax + NS + k] = v;
    }
    __syncthreads();
    if (warp == 0) {  // CTA partials (lane 0 writes all K, so thread 0's fence covers them)
      double v[K];
#pragma unroll
      for (int k = 0; k < NS; ++k) v[k] = warp_sum_down(lane < nw ? buf[lane * kRedMax + k] : 0.0);
#pragma unroll
      for (int k = 0; k < NM; ++k) v[NS + k] = warp_max_down(lane < nw ? buf[lane * kRedMax + NS + k] : -__builtin_huge_val());
      if (lane == 0)
#pragma unroll
        for (int k = 0; k < K; ++k) gp[blockIdx.x * kRedMax + k] = v[k];
    }
    const bool last = arrive(&last_flag);
    if (last && warp < K) {  // one warp per value, all values in parallel, CTA order fixed
      const int k = warp;
      const bool is_sum = k < NS;
      const int nb = gridDim.x;
      double part[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int b = lane + 32 * u;
        part[u] = b < nb ? __ldcg(gp + b * kRedMax + k) : (is_sum ? 0.0 : -__builtin_huge_val());
      }
      double acc = is_sum ? 0.0 : -__builtin_huge_val();
#pragma unroll
      for (int u = 0; u < 8; ++u) acc = is_sum ? acc + part[u] : fmax(acc, part[u]);
      for (int b = lane + 256; b < nb; b += 32) {
        const double x = __ldcg(gp + b * kRedMax + k);
        acc = is_sum ? acc + x : fmax(acc, x);
      }
      acc = is_sum ? warp_sum_down(acc) : warp_max_down(acc);
      if (lane == 0) __stcg(gr + k, acc);
    }
    if (last) __syncthreads();  // totals written before thread 0's release store
    release_or_wait(last);
#pragma unroll
    for (int k = 0; k < NS; ++k) s[k] = __ldcg(gr + k);
#pragma unroll
    for (int k = 0; k < NM; ++k) m[k] = __ldcg(gr + NS + k);
  }
};

}  // namespace nsd
