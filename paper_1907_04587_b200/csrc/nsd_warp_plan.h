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

// Per-env shared-memory layout, byte offsets: R (state/assembly) arrays, S (PCR
// operator) arrays, the staging area sized for R values (it holds R or S values),
// then the int lists.
struct Plan {
  int bq, brot, bu, biwi, bhi, bw, stg, rec, x, bx, gent_off, gent;
  int bytes;  // per env, 16-byte multiple
  template <class R, class S> static Plan make(int nb) {
    Plan p{};
    int o = 0;
    auto a = [&](int bytes) {
      const int off = o;
      o += (bytes + 15) & ~15;  // 16-byte aligned sub-arrays
      return off;
    };
    const int r = sizeof(R), sz = sizeof(S);
    p.bq = a(8 * nb * r);  // pos 3, quat 4, pad
    p.brot = a(9 * nb * r);
    p.bu = a(6 * nb * r);
    p.biwi = a(6 * nb * r);
    p.bhi = a(nb * r);     // 1 / (m + 0): H^-1 of the linear block (rigid dofs carry no shift)
    p.bw = a(6 * nb * sz);  // w = H^-1 J^T y of the operator
    p.stg = a(kStg * 32 * r);
    p.rec = a(rec_stride<S>() * 32 * sz);
    p.x = a(kRows * 32 * r);  // lane-private row vectors, [row][lane]
    p.bx = a(kRows * 32 * r);
    p.gent_off = a((nb + 1) * 4);  // per body: first entry; entries are staging offsets
    p.gent = a(64 * 4);            // (object * kStg + 6 * side)
    p.bytes = o;
    return p;
  }
};

}  // namespace wp
}  // namespace nsd
