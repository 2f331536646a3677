// Single-scene kernels (nsd_step, the newton_step boundary): one CTA for small
// scenes, a persistent cooperative grid for the FEM configs. Compiled twice: this
// TU (fp64 J/C coefficients, namespace nsdi::s64) and nsd_k_single32.cu (NSD_OP32=1:
// the fp32 mode's float coefficients, namespace nsdi::s32).
#ifndef NSD_OP32
#define NSD_OP32 0
#endif
#define NSD_ASM_NOINLINE 1
#include "nsd_plan.cuh"

#if NSD_OP32
#define NSD_SINGLE_NS s32
#else
#define NSD_SINGLE_NS s64
#endif

namespace nsdi {
namespace NSD_SINGLE_NS {

template <class R, bool kTets>
// 256 threads at most: the one CTA has the SM's register file to itself, so the
// engine runs without spills (128 registers at 512 threads spilled ~1 KB per thread:
// C1 0.417 -> 0.392 ms, C3 1.92 -> 1.75 ms per step at 256).
__global__ void __launch_bounds__(256) k_single_block(nsd::Topo<R> T, nsd::Work<R> W, nsd::Cfg cfg, nsd::StepOut out) {
  __shared__ double red[2 * 33 * nsd::kRedMax];
  nsd::BlockTeam t(red);
  nsd::newton_setup(t, T, W);
  t.sync();
  nsd::newton_solve<R, kTets>(t, T, W, cfg, out);
}

template <class R, bool kTets, int RPT>
__global__ void __launch_bounds__(kGridThreads) k_single_grid(nsd::Topo<R> T, nsd::Work<R> W, nsd::Cfg cfg, nsd::StepOut out,
                                                     double* gpart) {
  __shared__ double red[2 * 33 * nsd::kRedMax];
  nsd::GridTeam t(red, gpart);
#ifdef NSD_PROFILE_GRID
  if (out.ptime) t.prof = out.ptime + 8;
#endif
  nsd::newton_setup(t, T, W);
  t.sync();
  nsd::newton_solve<R, kTets, nsd::GridTeam, RPT>(t, T, W, cfg, out);
}

template <class R> int single_grid_blocks_per_sm(bool tets) {
  int per_sm = 0;
  if (tets)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_single_grid<R, true, 0>, kGridThreads, 0);
  else
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_single_grid<R, false, 0>, kGridThreads, 0);
  return per_sm;
}

template <class R>
cudaError_t launch_single_block(bool tets, int threads, cudaStream_t s, const nsd::Topo<R>& T, const nsd::Work<R>& W,
                                const nsd::Cfg& c, const nsd::StepOut& o) {
  if (tets)
    k_single_block<R, true><<<1, threads, 0, s>>>(T, W, c, o);
  else
    k_single_block<R, false><<<1, threads, 0, s>>>(T, W, c, o);
  return cudaGetLastError();
}

// mode: 0 memory-path PCR, 2 register-resident rows, -1 partitioned (smem bytes of
// dynamic shared memory per CTA, nsd_part.cuh)
template <class R>
cudaError_t launch_single_grid(bool tets, int mode, size_t smem, int blocks, cudaStream_t s, const nsd::Topo<R>& T,
                               const nsd::Work<R>& W, const nsd::Cfg& c, const nsd::StepOut& o, double* gpart) {
  nsd::Topo<R> t = T;
  nsd::Work<R> w = W;
  nsd::Cfg cf = c;
  nsd::StepOut so = o;
  void* args[] = {&t, &w, &cf, &so, &gpart};
  void* fn;
  if (mode < 0) {
    fn = tets ? (void*)k_single_grid<R, true, -1> : (void*)k_single_grid<R, false, -1>;
    const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  } else if (mode == 2) {
    fn = tets ? (void*)k_single_grid<R, true, 2> : (void*)k_single_grid<R, false, 2>;
    smem = 0;
  } else {
    fn = tets ? (void*)k_single_grid<R, true, 0> : (void*)k_single_grid<R, false, 0>;
    smem = 0;
  }
  return cudaLaunchCooperativeKernel(fn, dim3(blocks), dim3(kGridThreads), args, smem, s);
}

template int single_grid_blocks_per_sm<double>(bool);
template cudaError_t launch_single_block<double>(bool, int, cudaStream_t, const nsd::Topo<double>&,
                                                 const nsd::Work<double>&, const nsd::Cfg&, const nsd::StepOut&);
template cudaError_t launch_single_grid<double>(bool, int, size_t, int, cudaStream_t, const nsd::Topo<double>&,
                                                const nsd::Work<double>&, const nsd::Cfg&, const nsd::StepOut&, double*);

}  // namespace NSD_SINGLE_NS
}  // namespace nsdi
