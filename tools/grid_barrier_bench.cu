// Microbenchmark of the grid-wide all-reduce alone (no PCR work): the cost floor of
// one GridTeam::reduce_sum on 148 co-resident CTAs, against variants of the arrival.
//   nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_1907_04587_b200/csrc \
//        grid_barrier_bench.cu -o _grid_barrier_bench && ./_grid_barrier_bench
// Variants (arrival / wait of GridTeam::sync, the rest of the reduction unchanged):
//   0  product: thread 0 atom.acq_rel on one count, ld.acquire spin
//   1  16 counts 1 KB apart: thread 0 red.release on count b % 16, lanes 0..15 of warp 0
//      spin with ld.acquire on one count each
//   2  tree: 16 groups; the last arriver of a group (atom.acq_rel return value)
//      arrives on the root; thread 0 spins on the root only
//   3  explicit fences: fence.acq_rel; atom.relaxed; ld.relaxed spin; fence.acq_rel
//   4  legacy: membar.gl; atom; volatile spin; membar.gl (cooperative-groups style)
//   5  the product barrier alone (no partials written or read): the barrier floor
//   6  no grid barrier at all (CTA-local sums only): the local floor
//   7, 8  the product barrier with the partials replicated 4 / 8 times (CTA b reads
//      copy b % R): R times fewer readers per L2 line
#include <cooperative_groups.h>
#include <cstdio>
#include <vector>

#include "nsd_team.cuh"

namespace {

constexpr int kStride = 256;  // unsigneds between counts (1 KB)

template <int V> struct Team : nsd::GridTeam {
  unsigned* ctr;
  __device__ Team(double* red, double* gp, unsigned* c) : nsd::GridTeam(red, gp), ctr(c) {}
  __device__ __forceinline__ void sync() {
    if constexpr (V == 0 || V == 5 || V == 7 || V == 8) {
      nsd::GridTeam::sync();
      return;
    }
    if constexpr (V == 6) {
      __syncthreads();
      return;
    }
    __syncthreads();
    ++epoch;
    const int nb = gridDim.x;
    if constexpr (V == 1) {
      if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        if (lane == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr + (blockIdx.x % 16) * kStride) : "memory");
        if (lane < 16) {
          const unsigned target = epoch * static_cast<unsigned>((nb - lane + 15) / 16);
          unsigned v;
          do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr + lane * kStride) : "memory");
          } while (static_cast<int>(v - target) < 0);
        }
        __syncwarp();
      }
    } else if constexpr (V == 3 || V == 4) {
      if (threadIdx.x == 0) {
        if constexpr (V == 3) asm volatile("fence.acq_rel.gpu;" ::: "memory");
        else asm volatile("membar.gl;" ::: "memory");
        unsigned prev;
        if constexpr (V == 3) asm volatile("atom.relaxed.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(ctr) : "memory");
        else prev = atomicAdd(ctr, 1u);
        const unsigned target = epoch * nb;
        if (prev + 1u != target) {
          unsigned v;
          do {
            if constexpr (V == 3) asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
            else v = *reinterpret_cast<volatile unsigned*>(ctr);
          } while (static_cast<int>(v - target) < 0);
        }
        if constexpr (V == 3) asm volatile("fence.acq_rel.gpu;" ::: "memory");
        else asm volatile("membar.gl;" ::: "memory");
      }
    } else {
      if (threadIdx.x == 0) {
        const int g = blockIdx.x % 16;
        const unsigned gsize = static_cast<unsigned>((nb - g + 15) / 16);
        unsigned prev;
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(ctr + (1 + g) * kStride) : "memory");
        if (prev + 1u == epoch * gsize)
          asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
        const unsigned target = epoch * 16u;
        unsigned v;
        do {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
        } while (static_cast<int>(v - target) < 0);
      }
    }
    __syncthreads();
  }
};

template <int V> __global__ void __launch_bounds__(256) k_bench(double* gpart, unsigned* ctr, int iters, double* out) {
  __shared__ double red[2 * 33 * nsd::kRedMax];
  Team<V> t(red, gpart, ctr);
  double acc = 0.0;
  for (int i = 0; i < iters; ++i) {
    double s[2] = {static_cast<double>(threadIdx.x + i), acc * 1e-30};
    // the reduction of nsd_team.cuh with this variant's barrier
    double* buf = t.red + t.parity * (33 * nsd::kRedMax);
    constexpr int kRep = V == 7 ? 4 : (V == 8 ? 8 : 1);
    double* gp = t.gpart + t.parity * (gridDim.x * nsd::kRedMax);
    double* gx = t.gpart + 2 * gridDim.x * nsd::kRedMax + 64 + t.parity * (kRep * gridDim.x * 2);  // replicas
    t.parity ^= 1;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int k = 0; k < 2; ++k) {
      const double v = nsd::warp_sum_down(s[k]);
      if (lane == 0) buf[warp * nsd::kRedMax + k] = v;
    }
    __syncthreads();
    if (V != 5 && warp == 0) {
      double v0 = nsd::warp_sum_down(lane < nw ? buf[lane * nsd::kRedMax] : 0.0);
      double v1 = nsd::warp_sum_down(lane < nw ? buf[lane * nsd::kRedMax + 1] : 0.0);
      if (kRep == 1) {
        if (lane == 0) {
          gp[0 * gridDim.x + blockIdx.x] = v0;
          gp[1 * gridDim.x + blockIdx.x] = v1;
        }
      } else if (lane < kRep) {  // replica `lane`
        gx[(lane * 2 + 0) * gridDim.x + blockIdx.x] = v0;
        gx[(lane * 2 + 1) * gridDim.x + blockIdx.x] = v1;
      }
    }
    t.sync();
    if (V != 5 && warp < 2) {
      double part[8];  // all loads in flight at once, as GridTeam::red_impl
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int bb = lane + 32 * u;
        const double* src = kRep == 1 ? gp + warp * gridDim.x : gx + ((blockIdx.x % kRep) * 2 + warp) * gridDim.x;
        part[u] = bb < (int)gridDim.x ? __ldcg(src + bb) : 0.0;
      }
      double a = 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u) a += part[u];
      a = nsd::warp_sum_down(a);
      if (lane == 0) buf[32 * nsd::kRedMax + warp] = a;
    }
    __syncthreads();
    acc += buf[32 * nsd::kRedMax] + buf[32 * nsd::kRedMax + 1];
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) *out = acc;
}

template <int V> float run(int nb, int iters, double* gpart, unsigned* ctr, size_t ctr_bytes, double* out) {
  cudaMemset(ctr, 0, ctr_bytes);
  cudaMemset(gpart, 0, sizeof(double) * (nsd::grid_scratch_doubles(nb) + 64 + 2 * 8 * nb * 2));
  void* args[] = {&gpart, &ctr, &iters, &out};
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  cudaLaunchCooperativeKernel((void*)k_bench<V>, dim3(nb), dim3(256), args, 0, 0);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) std::printf("error %s\n", cudaGetErrorString(e));
  return ms;
}

}  // namespace

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 4000;
  double *gpart, *out;
  unsigned* ctr;
  const size_t ctr_bytes = sizeof(unsigned) * kStride * 17;
  cudaMalloc(&gpart, sizeof(double) * (nsd::grid_scratch_doubles(320) + 64 + 2 * 8 * 320 * 2));
  cudaMalloc(&ctr, ctr_bytes);
  cudaMalloc(&out, sizeof(double));
  for (int nb : {sms, sms / 2}) {
    for (int rep = 0; rep < 2; ++rep) {
      const float t0 = run<0>(nb, iters, gpart, ctr, ctr_bytes, out);
      const float t1 = run<1>(nb, iters, gpart, ctr, ctr_bytes, out);
      const float t2 = run<2>(nb, iters, gpart, ctr, ctr_bytes, out);
      const float t3 = run<3>(nb, iters, gpart, ctr, ctr_bytes, out);
      const float t4 = run<4>(nb, iters, gpart, ctr, ctr_bytes, out);
      const float t5 = run<5>(nb, iters, gpart, ctr, ctr_bytes, out);
      const float t6 = run<6>(nb, iters, gpart, ctr, ctr_bytes, out);
      const float t7 = run<7>(nb, iters, gpart, ctr, ctr_bytes, out);
      const float t8 = run<8>(nb, iters, gpart, ctr, ctr_bytes, out);
      std::printf("CTAs %d: us per 2-value grid reduction: product %.3f  16-counts %.3f  tree %.3f  fences %.3f  "
                  "legacy %.3f | barrier only %.3f  local only %.3f | replicas x4 %.3f x8 %.3f\n",
                  nb, 1000.f * t0 / iters, 1000.f * t1 / iters, 1000.f * t2 / iters, 1000.f * t3 / iters,
                  1000.f * t4 / iters, 1000.f * t5 / iters, 1000.f * t6 / iters, 1000.f * t7 / iters,
                  1000.f * t8 / iters);
    }
  }
  return 0;
}
