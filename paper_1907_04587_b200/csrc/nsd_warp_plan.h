// Shared-memory plan of the warp-per-environment batch solver (nsd_warp.cuh),
// kept apart so the host layer and the other kernel units do not depend on the
// solver's device code.
#pragma once

namespace nsd {
namespace wp {

constexpr int kRows = 5;   // rows per object (joint <= 5, contact 3)
constexpr int kRec = 21;   // record: arm_a 3, arm_b 3, 5 row directions x 3
constexpr int kStg = 14;   // staging stride: a.lin a.ang b.lin b.ang (12) + pad
constexpr int kWPhases = 14;  // NSD_PHASE_TIMING counters of the warp solver

// Record stride per object (elements): 21 values padded so that 16-byte loads by
// 8 consecutive lanes hit distinct bank quads (fp64 22 = 44 words = 12 mod 32;
// fp32 28 words = 28 mod 32).
template <class R> __host__ __device__ constexpr int rec_stride() { return sizeof(R) == 8 ? 22 : 28; }

// Per-env shared-memory layout (element offsets; R part then int part).
struct Plan {
  int bq, brot, bu, biwi, bhi, bw, stg, rec, x, bx, nR;  // R elements
  int gent_off, gent, nI;                                      // int elements after the R part
  int bytes;                                                   // per env, 16-byte multiple
  template <class R> static Plan make(int nb) {
    Plan p{};
    int o = 0;
    auto a = [&](int n) {
      const int off = o;
      o += (n + 3) & ~3;  // 16-byte aligned sub-arrays (fp32 and fp64)
      return off;
    };
    p.bq = a(8 * nb);  // pos 3, quat 4, pad
    p.brot = a(9 * nb);
    p.bu = a(6 * nb);
    p.biwi = a(6 * nb);
    p.bhi = a(nb);     // 1 / (m + 0): H^-1 of the linear block (rigid dofs carry no shift)
    p.bw = a(6 * nb);  // w = H^-1 J^T y
    p.stg = a(kStg * 32);
    p.rec = a(rec_stride<R>() * 32);
    p.x = a(kRows * 32);  // lane-private row vectors, [row][lane]
    p.bx = a(kRows * 32);
    p.nR = o;
    p.gent_off = 0;  // per body: first entry; entries are staging offsets (object * kStg + 6 * side)
    p.gent = (nb + 1 + 3) & ~3;
    p.nI = p.gent + 64;
    p.bytes = ((o * (int)sizeof(R) + 15) & ~15) + ((p.nI * 4 + 15) & ~15);
    return p;
  }
};

}  // namespace wp
}  // namespace nsd
