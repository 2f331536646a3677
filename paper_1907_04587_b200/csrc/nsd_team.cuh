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

#include "nsd_math.cuh"  // NSD_CHECK

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

// Grid team: one cooperative launch, one CTA per SM (<= 320 CTAs). Barrier: every
// CTA arrives on a global count that only grows within a launch and spins until it
// reaches this barrier's target. All-reduce: each CTA publishes its partials, passes
// the barrier, then sums every CTA's partials itself, in CTA order, with the same
// code in every CTA — so every member gets the identical bits (deterministic,
// team-uniform branches). Partials are stored value-major (one value's partials of
// all CTAs contiguous: 37 sectors per value for 148 CTAs), double-buffered by parity.
// Measured history (C2 FEM): CG grid sync + value-by-value re-read
// 18.0 ms/step; "last CTA reduces and releases a generation flag" 11.1 ms; this
// scheme 8.0 ms (two L2 round trips fewer per reduction); partitioned PCR 5.0 ms.
// Tried and slower (profiles/r2_grid_barrier_ab.txt): flag-in-data partials (each
// partial carries its epoch, no count; every CTA polling every CTA's words hammers
// the same L2 lines: 15.4 vs 9.0 us per CR iteration), and 16 arrival counts 1 KB
// apart polled by the lanes of warp 0 with one acquire fence (6.0 vs 5.0 ms/step).
// The partitioned PCR also tried ONE grid reduction per CR iteration, with the
// shared blocks' partials exchanged point to point (release flag per CTA, acquire
// polls of the neighbour CTAs only): 5.5 vs 5.0 ms/step — a neighbour handshake
// costs as much as the grid barrier (release, flag, poll and acquire are ~3 L2
// round trips either way; measured ~4,600 cycles per grid reduction on C2 with the
// CTAs' compute balanced to 4 %).
// Double buffering suffices: a CTA can write reduction n + 2's partials (same
// parity as n) only after passing reduction n + 1's barrier, which every CTA
// reaches only after it finished reading reduction n's partials.
constexpr int kGridMaxCtas = 320;
// Global scratch (doubles): [2 x nb x kRedMax partials][2 x kRedMax unused][count, unused].
__host__ __device__ constexpr size_t grid_scratch_count_off(int nb) { return 2 * (size_t)nb * kRedMax + 2 * kRedMax; }
__host__ __device__ constexpr size_t grid_scratch_doubles(int nb) { return grid_scratch_count_off(nb) + 2; }
// what the host zeroes before every launch: the count
__host__ __device__ constexpr size_t grid_scratch_reset_off(int nb) { return grid_scratch_count_off(nb); }

struct GridTeam {
  double* red;    // shared: 2 * (33 * kRedMax)
  double* gpart;  // global partials
  unsigned* bar;  // [0] arrival count
  int parity;
  unsigned epoch;
  // NSD_PHASE_TIMING diagnostics: CTA 0 thread 0's cycles per reduction stage
  // (local sums, partial store, arrival atomic, spin, partial sums, tail), or null
  unsigned long long* prof = nullptr;
  long long pt = 0;
  __device__ __forceinline__ void pmark(int k) {
#ifdef NSD_PROFILE_GRID  // compile-time: the counters' register and branch cost is not free in the PCR loop
    if (prof && blockIdx.x == 0 && threadIdx.x == 0) {
      const long long t = clock64();
      if (k >= 0) prof[k] += static_cast<unsigned long long>(t - pt);
      pt = t;
    }
#else
    (void)k;
#endif
  }
  __device__ GridTeam(double* smem_red, double* global_part)
      : red(smem_red), gpart(global_part),
        bar(reinterpret_cast<unsigned*>(global_part + grid_scratch_count_off(gridDim.x))), parity(0), epoch(0) {}
  __device__ __forceinline__ int rank() const { return blockIdx.x * blockDim.x + threadIdx.x; }
  __device__ __forceinline__ int size() const { return gridDim.x * blockDim.x; }
  static __device__ __forceinline__ int part_idx(int b, int k) { return k * gridDim.x + b; }

  // Arrive and wait for every CTA. Thread 0's acq_rel atomic publishes the CTA's
  // writes (ordered before it by the __syncthreads) and its acquire loads see
  // every other CTA's; the closing __syncthreads extends that to the whole CTA.
  // CTAs already past this barrier may arrive at the next one before a slow
  // spinner reads the count, hence the signed-distance test.
  __device__ __forceinline__ void sync() {
    __syncthreads();
    ++epoch;
    if (threadIdx.x == 0) {
      const bool timed = pt != 0;  // inside a reduction (plain barriers are not profiled)
      if (timed) pmark(1);
      unsigned prev;
      asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(bar) : "memory");
      // no CTA can arrive at the next barrier before this one completes
      NSD_CHECK(static_cast<int>(prev + 1u - epoch * gridDim.x) <= 0);
      if (timed) pmark(2);
      const unsigned target = epoch * gridDim.x;
      if (prev + 1u != target) {
        unsigned c;
        do {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(c) : "l"(bar) : "memory");
        } while (static_cast<int>(c - target) < 0);
      }
      if (timed) pmark(3);
    }
    __syncthreads();
  }
  template <int NS> __device__ __forceinline__ void reduce_sum(double (&s)[NS]) {
    red_impl<NS, 0>(s, nullptr, NoSide{});
  }
  struct NoSide {
    __device__ __forceinline__ void operator()(int, int) const {}
  };
  template <int NS, int NM>
  __device__ __forceinline__ void reduce(double (&s)[NS], double (&m)[NM]) {
    red_impl<NS, NM>(s, m, NoSide{});
  }
  // side(first, n): work for the threads of the warps that do not sum partials, run
  // after the barrier concurrently with the partial sums (threads first, first + 1,
  // ... of n); its shared-memory writes are visible when reduce returns.
  template <int NS, class F>
  __device__ __forceinline__ void reduce_sum_side(double (&s)[NS], F&& side) {
    red_impl<NS, 0>(s, nullptr, side);
  }
  // sums s[0..NS), maxima m[0..NM) (m may be null when NM == 0)
  template <int NS, int NM, class F>
  __device__ __forceinline__ void red_impl(double* s, double* m, F&& side) {
    constexpr int K = NS + NM;
    static_assert(K <= kRedMax && K > 0, "1..kRedMax values per reduction");
    pmark(-1);
    double* buf = red + parity * (33 * kRedMax);
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
    const int nb = gridDim.x;
    double* gp = gpart + parity * (nb * kRedMax);
    parity ^= 1;
    if (warp == 0) {  // CTA partials
      double v[K > 0 ? K : 1];
#pragma unroll
      for (int k = 0; k < NS; ++k) v[k] = warp_sum_down(lane < nw ? buf[lane * kRedMax + k] : 0.0);
#pragma unroll
      for (int k = 0; k < NM; ++k) v[NS + k] = warp_max_down(lane < nw ? buf[lane * kRedMax + NS + k] : -__builtin_huge_val());
      if (lane == 0)
#pragma unroll
        for (int k = 0; k < K; ++k) gp[part_idx(blockIdx.x, k)] = v[k];
    }
    sync();
    if (warp >= K) side(threadIdx.x - 32 * K, static_cast<int>(blockDim.x) - 32 * K);
    if (warp < K) {  // one warp per value, all values in parallel, CTA order fixed
      const int k = warp;
      const bool is_sum = k < NS;
      double part[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int b = lane + 32 * u;
        part[u] = b < nb ? __ldcg(gp + part_idx(b, k)) : (is_sum ? 0.0 : -__builtin_huge_val());
      }
      double acc = is_sum ? 0.0 : -__builtin_huge_val();
#pragma unroll
      for (int u = 0; u < 8; ++u) acc = is_sum ? acc + part[u] : fmax(acc, part[u]);
      for (int b = lane + 256; b < nb; b += 32) {
        const double x = __ldcg(gp + part_idx(b, k));
        acc = is_sum ? acc + x : fmax(acc, x);
      }
      acc = is_sum ? warp_sum_down(acc) : warp_max_down(acc);
      if (lane == 0) buf[32 * kRedMax + k] = acc;
    }
    pmark(4);
    __syncthreads();
    pmark(5);
#ifdef NSD_PROFILE_GRID
    pt = 0;
#endif
#pragma unroll
    for (int k = 0; k < NS; ++k) s[k] = buf[32 * kRedMax + k];
#pragma unroll
    for (int k = 0; k < NM; ++k) m[k] = buf[32 * kRedMax + NS + k];
  }
};

}  // namespace nsd
