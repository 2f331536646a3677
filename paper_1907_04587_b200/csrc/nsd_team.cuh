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

// Grid team: one cooperative launch, one CTA per SM (<= 320 CTAs). Every CTA
// sums all CTAs' partials itself, in CTA order, with the same code in every CTA —
// so every member gets the identical bits (deterministic, team-uniform branches).
//
// Arrival is flag-in-data (NSD_GRID_LL, default): a CTA publishes each partial as
// one 16-byte store of two 8-byte words, (epoch << 32 | low 32 bits) and
// (epoch << 32 | high 32 bits), after a release fence. Readers poll the words of
// all CTAs until every word carries the current epoch; the data arrive with the
// flags, so one L2 round trip after the last writer ends the reduction. There is
// no arrival counter: no 148-way atomic serialisation at one L2 slice and no
// separate read of the partials after the count completes. Each 8-byte word is
// single-copy atomic, so a word with the current epoch holds the current bits.
// Plain barriers (sync) publish one epoch word per CTA; warp 0 polls all of them.
//   Partials are double-buffered by parity. A CTA can write reduction n + 2's
// words (same parity as n) only after passing reduction n + 1, which every CTA
// reaches only after it finished reading reduction n's words; stale words carry
// older epochs and are never accepted. Epochs restart at 1 every launch: the host
// zeroes the flag words before each launch (grid_scratch_reset).
//   NSD_GRID_LL=0 builds the previous scheme (one acq_rel arrival on a monotonic
// count, then the value-major partials are read): C2 8.9 us per CR iteration.
// Measured history (C2 FEM): CG grid sync + value-by-value re-read
// 18.0 ms/step; "last CTA reduces and releases a generation flag" 11.1 ms; count
// + every CTA reduces 8.0 ms; partitioned PCR 5.4 ms.
#ifndef NSD_GRID_LL
#define NSD_GRID_LL 0
#endif
constexpr int kGridMaxCtas = 320;
// Global scratch (doubles): [2 x nb x kRedMax partials][2 x kRedMax unused][count, unused]
// then, 16-byte aligned, the flag-in-data words [2 parity][kRedMax][nb][2] and the
// barrier words [nb].
__host__ __device__ constexpr size_t grid_scratch_count_off(int nb) { return 2 * (size_t)nb * kRedMax + 2 * kRedMax; }
__host__ __device__ constexpr size_t grid_scratch_ll_off(int nb) { return (grid_scratch_count_off(nb) + 2 + 1) & ~size_t(1); }
__host__ __device__ constexpr size_t grid_scratch_doubles(int nb) {
  return grid_scratch_ll_off(nb) + 4 * (size_t)kRedMax * nb + nb;
}
// what the host zeroes before every launch: [count .. end)
__host__ __device__ constexpr size_t grid_scratch_reset_off(int nb) { return grid_scratch_count_off(nb); }

__device__ __forceinline__ void ll_fence() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void ll_put(unsigned long long* p, double v, unsigned e) {
  const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
  const unsigned long long hi = static_cast<unsigned long long>(e) << 32;
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(hi | (b & 0xffffffffull)), "l"(hi | (b >> 32))
               : "memory");
}
__device__ __forceinline__ void ll_get(const unsigned long long* p, unsigned long long& w0, unsigned long long& w1) {
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(w0), "=l"(w1) : "l"(p) : "memory");
}

struct GridTeam {
  double* red;    // shared: 2 * (33 * kRedMax)
  double* gpart;  // global partials
  unsigned* bar;  // [0] arrival count
  unsigned long long* ll;     // flag-in-data partials [2][kRedMax][nb][2]
  unsigned long long* lflag;  // barrier words [nb]
  int parity;
  unsigned epoch;
  __device__ GridTeam(double* smem_red, double* global_part)
      : red(smem_red), gpart(global_part),
        bar(reinterpret_cast<unsigned*>(global_part + grid_scratch_count_off(gridDim.x))),
        ll(reinterpret_cast<unsigned long long*>(global_part + grid_scratch_ll_off(gridDim.x))),
        lflag(ll + 4 * (size_t)kRedMax * gridDim.x), parity(0), epoch(0) {}
  __device__ __forceinline__ int rank() const { return blockIdx.x * blockDim.x + threadIdx.x; }
  __device__ __forceinline__ int size() const { return gridDim.x * blockDim.x; }
  static __device__ __forceinline__ int part_idx(int b, int k) { return k * gridDim.x + b; }

  // Arrive and wait for every CTA. The release (fence + flag store by thread 0 after
  // the __syncthreads) publishes the CTA's writes; warp 0's acquire (fence after
  // the polls) sees every other CTA's, and the closing __syncthreads extends that
  // to the whole CTA. CTAs already past this barrier may publish the next epoch
  // before a slow poller reads the word, hence the signed-distance test.
  __device__ __forceinline__ void sync() {
    __syncthreads();
    ++epoch;
#if NSD_GRID_LL
    if (threadIdx.x < 32) {
      const int lane = threadIdx.x, nb = gridDim.x;
      if (lane == 0) {
        ll_fence();
        asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(lflag + blockIdx.x),
                     "l"(static_cast<unsigned long long>(epoch))
                     : "memory");
      }
      bool ok;
      do {
        ok = true;
#pragma unroll
        for (int u = 0; u < kGridMaxCtas / 32; ++u) {
          const int b = lane + 32 * u;
          if (b < nb) {
            unsigned long long f;
            asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(f) : "l"(lflag + b) : "memory");
            ok &= static_cast<int>(static_cast<unsigned>(f) - epoch) >= 0;
          }
        }
      } while (!__all_sync(0xffffffffu, ok));
      ll_fence();
    }
#else
    if (threadIdx.x == 0) {
      unsigned prev;
      asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(bar) : "memory");
      const unsigned target = epoch * gridDim.x;
      if (prev + 1u != target) {
        unsigned c;
        do {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(c) : "l"(bar) : "memory");
        } while (static_cast<int>(c - target) < 0);
      }
    }
#endif
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
#if NSD_GRID_LL
    ++epoch;
    unsigned long long* lp = ll + (size_t)parity * kRedMax * nb * 2;
    parity ^= 1;
    if (warp == 0) {  // CTA partials, published with the epoch after a release fence
      double v[K > 0 ? K : 1];
#pragma unroll
      for (int k = 0; k < NS; ++k) v[k] = warp_sum_down(lane < nw ? buf[lane * kRedMax + k] : 0.0);
#pragma unroll
      for (int k = 0; k < NM; ++k) v[NS + k] = warp_max_down(lane < nw ? buf[lane * kRedMax + NS + k] : -__builtin_huge_val());
      if (lane == 0) {
        ll_fence();
#pragma unroll
        for (int k = 0; k < K; ++k) ll_put(lp + 2 * ((size_t)k * nb + blockIdx.x), v[k], epoch);
      }
    }
    // warps < K poll (and then sum) value k of every CTA; the side warps wait on
    // named barrier 1 for warp 0's acquire
    constexpr int kU = kGridMaxCtas / 32;
    if (warp < K) {
      const int k = warp;
      const bool is_sum = k < NS;
      const unsigned long long* src = lp + 2 * (size_t)k * nb;
      double part[kU];
      bool ok;
      do {
        ok = true;
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int b = lane + 32 * u;
          if (b < nb) {
            unsigned long long w0, w1;
            ll_get(src + 2 * b, w0, w1);
            ok &= (static_cast<unsigned>(w0 >> 32) == epoch) & (static_cast<unsigned>(w1 >> 32) == epoch);
            part[u] = __longlong_as_double(static_cast<long long>((w1 << 32) | (w0 & 0xffffffffull)));
          } else {
            part[u] = is_sum ? 0.0 : -__builtin_huge_val();
          }
        }
      } while (!__all_sync(0xffffffffu, ok));
      ll_fence();
      if (warp == 0 && nw > K) asm volatile("bar.arrive 1, %0;" ::"r"(32 * (nw - K + 1)) : "memory");
      double acc = is_sum ? 0.0 : -__builtin_huge_val();
#pragma unroll
      for (int u = 0; u < kU; ++u) acc = is_sum ? acc + part[u] : fmax(acc, part[u]);
      acc = is_sum ? warp_sum_down(acc) : warp_max_down(acc);
      if (lane == 0) buf[32 * kRedMax + k] = acc;
    } else {
      asm volatile("bar.sync 1, %0;" ::"r"(32 * (nw - K + 1)) : "memory");
      side(threadIdx.x - 32 * K, static_cast<int>(blockDim.x) - 32 * K);
    }
#else
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
#endif
    __syncthreads();
#pragma unroll
    for (int k = 0; k < NS; ++k) s[k] = buf[32 * kRedMax + k];
#pragma unroll
    for (int k = 0; k < NM; ++k) m[k] = buf[32 * kRedMax + NS + k];
  }
};

}  // namespace nsd
