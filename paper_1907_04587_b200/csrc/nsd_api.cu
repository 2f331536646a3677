// C-ABI implementation (include/nsdyn_gpu.h): handles, device memory, kernels.
//
//   k_single_block / k_single_grid  one scene, nsd_step (newton_step boundary)
//   k_batch_sub / k_batch_block     many environments, nsd_batch_step
//                                   (device narrow phase + newton_step per env)
//   k_batch_warp                    many rigid environments: one warp per env,
//                                   after k_batch_sub's narrow-phase launch
#include "nsdyn_gpu.h"

#include "nsd_plan.cuh"

#include <nvtx3/nvToolsExt.h>

#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace {

using namespace nsdi;

thread_local std::string g_err;

// NVTX range (nsys / ncu --nvtx): the host phases of a step around its launches. The
// Newton phases run inside one persistent launch; their device time comes from the
// in-kernel clock64 counters (NSD_PHASE_TIMING, nsd_batch_profile).
struct Nvtx {
  explicit Nvtx(const char* name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
  Nvtx(const Nvtx&) = delete;
  Nvtx& operator=(const Nvtx&) = delete;
};
// Consecutive sub-ranges of one scope (each start() closes the previous one).
// NVTX range per host phase of a step; with acc set (NSD_HOST_TIMING) it also sums
// each phase's wall time (ms) into acc[k], k = the phase's ordinal.
struct NvtxPhase {
  bool open = false;
  double* acc = nullptr;
  int k = -1;
  std::chrono::steady_clock::time_point t0;
  void stamp() {
    if (acc && k >= 0) acc[k] += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (acc) t0 = std::chrono::steady_clock::now();
    ++k;
  }
  void start(const char* name) {
    if (open) nvtxRangePop();
    stamp();
    nvtxRangePushA(name);
    open = true;
  }
  ~NvtxPhase() {
    if (open) nvtxRangePop();
    stamp();
  }
};

struct NsdError : std::runtime_error {
  int code;
  NsdError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define NSD_CK(call)                                                                           \
  do {                                                                                         \
    cudaError_t e_ = (call);                                                                   \
    if (e_ != cudaSuccess)                                                                     \
      throw NsdError(NSD_CUDA_ERROR, std::string(#call) + ": " + cudaGetErrorString(e_));      \
  } while (0)

template <class F> int guarded(F&& f) {
  try {
    return f();
  } catch (const NsdError& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return NSD_INVALID;
  }
}

// Device buffer (raw bytes).
struct DBuf {
  void* p = nullptr;
  size_t n = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() {
    if (p) cudaFree(p);
  }
  // Grows by at least 1.5x: a contact count creeping up step by step must not
  // re-allocate (cudaFree synchronises the device) on every step.
  void alloc(size_t bytes) {
    if (bytes <= n && p) return;
    if (p) cudaFree(p);
    p = nullptr;
    const size_t want = std::max<size_t>(std::max<size_t>(bytes, 16), n + n / 2);
    n = 0;
    NSD_CK(cudaMalloc(&p, want));
    n = want;
  }
  template <class T> T* as(size_t off_elems = 0) const { return static_cast<T*>(p) + off_elems; }
};

// Pinned host staging.
struct HBuf {
  void* p = nullptr;
  size_t n = 0;
  ~HBuf() {
    if (p) cudaFreeHost(p);
  }
  // Same 1.5x growth as DBuf: pinned (de)allocation costs milliseconds.
  void alloc(size_t bytes) {
    if (bytes <= n && p) return;
    if (p) cudaFreeHost(p);
    p = nullptr;
    const size_t want = std::max<size_t>(std::max<size_t>(bytes, 16), n + n / 2);
    n = 0;
    NSD_CK(cudaMallocHost(&p, want));
    n = want;
  }
};

// Bump allocator over a byte layout (256-byte aligned sub-arrays).
struct Layout {
  size_t bytes = 0;
  template <class T> size_t add(size_t count) {
    const size_t off = (bytes + 255) & ~size_t(255);
    bytes = off + sizeof(T) * std::max<size_t>(count, 1);
    return off;
  }
};

nsd::Cfg to_cfg(const nsd_config& c) {
  nsd::Cfg o;
  o.newton_iterations = c.newton_iterations;
  o.step_fraction = c.step_fraction;
  o.epsilon_reg = c.epsilon_reg;
  o.geometric_stiffness = c.geometric_stiffness;
  o.r_strategy = c.r_strategy;
  o.ncp_kind = c.ncp_kind;
  o.linear_max_iterations = c.linear_max_iterations;
  o.linear_tolerance = c.linear_tolerance;
  o.preconditioner = c.preconditioner;
  o.newton_tolerance = c.newton_tolerance;
  o.line_search = c.line_search;
  o.linear_method = c.linear_method;
  return o;
}

void check_cfg(const nsd_config& c) {
  if (c.precision != NSD_FP32 && c.precision != NSD_FP64) throw NsdError(NSD_INVALID, "precision must be 0 or 1");
  if (c.linear_method < 0 || c.linear_method > 3)
    throw NsdError(NSD_INVALID, "linear_method must be 0 (Jacobi), 1 (Gauss-Seidel), 2 (PCG) or 3 (PCR)");
  if (c.linear_max_iterations < 1) throw NsdError(NSD_INVALID, "solve_linear: max_iterations < 1");
  if (c.newton_iterations < 0) throw NsdError(NSD_INVALID, "newton_iterations < 0");
  if (c.r_strategy < 0 || c.r_strategy > 2 || c.ncp_kind < 0 || c.ncp_kind > 1 || c.preconditioner < 0 ||
      c.preconditioner > 1)
    throw NsdError(NSD_INVALID, "config enum out of range");
}

// ------------------------------------------------------------------ host topology preprocessing

// Inverse of the 6x6 isotropic stiffness by Gauss-Jordan with partial pivoting
// (the linear material's compliance, materials.cpp:121,153), same elimination
// order as the CPU oracle's restatement so both sides start from equal bits.
void inverse6_h(const double (&k)[6][6], double (&o)[6][6]) {
  double a[6][12];
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j < 12; ++j) a[i][j] = j < 6 ? k[i][j] : (j - 6 == i ? 1.0 : 0.0);
  for (int c = 0; c < 6; ++c) {
    int piv = c;
    for (int r = c + 1; r < 6; ++r)
      if (std::abs(a[r][c]) > std::abs(a[piv][c])) piv = r;
    if (piv != c)
      for (int j = 0; j < 12; ++j) std::swap(a[c][j], a[piv][j]);
    const double d = a[c][c];
    for (int j = 0; j < 12; ++j) a[c][j] /= d;
    for (int r = 0; r < 6; ++r) {
      if (r == c) continue;
      const double f = a[r][c];
      for (int j = 0; j < 12; ++j) a[r][j] -= f * a[c][j];
    }
  }
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j < 6; ++j) o[i][j] = a[i][j + 6];
}

void body_blocks_h(const HostTopo& T, int b, int& lin, int& ang) {
  if (b < 0) {
    lin = ang = -1;
    return;
  }
  lin = T.bdof[b] / 3;
  ang = T.btype[b] == 1 ? lin + 1 : -1;
}

HostTopo preprocess(const nsd_topology& tp) {
  HostTopo T;
  if (tp.n_bodies < 0 || tp.n_joints < 0 || tp.n_tets < 0) throw NsdError(NSD_INVALID, "negative counts");
  T.nb = tp.n_bodies;
  T.nj = tp.n_joints;
  T.nt = tp.n_tets;
  for (int b = 0; b < T.nb; ++b) {
    const int ty = tp.body_type[b];
    if (ty != 0 && ty != 1) throw NsdError(NSD_INVALID, "body type must be 0 or 1");
    if (!(tp.body_mass[b] > 0.0)) throw NsdError(NSD_INVALID, "body mass must be positive");
    T.btype.push_back(ty);
    T.bdof.push_back(T.ndof);
    T.bcoord.push_back(T.ncoord);
    T.ndof += ty ? 6 : 3;
    T.ncoord += ty ? 7 : 3;
    T.bmass.push_back(tp.body_mass[b]);
    for (int k = 0; k < 9; ++k) T.binertia.push_back(ty ? tp.body_inertia[9 * b + k] : (k % 4 == 0 ? 1.0 : 0.0));
    T.d3_body.push_back(b);
    T.d3_kind.push_back(ty ? nsd::kRigidLin : nsd::kParticleLin);
    if (ty) {
      T.d3_body.push_back(b);
      T.d3_kind.push_back(nsd::kRigidAng);
    }
  }
  T.nd3 = T.ndof / 3;
  int row = 0;
  for (int j = 0; j < T.nj; ++j) {
    const int k = tp.joint_kind[j];
    if (k < 0 || k > 3) throw NsdError(NSD_INVALID, "joint kind out of range");
    const int a = tp.joint_body[2 * j], b = tp.joint_body[2 * j + 1];
    if (a >= T.nb || b >= T.nb || a < -1 || b < -1) throw NsdError(NSD_INVALID, "joint references invalid body");
    T.jkind.push_back(k);
    T.jbody.push_back(a);
    T.jbody.push_back(b);
    T.jrow.push_back(row);
    row += nsd::joint_nrows(k);
    for (int i = 0; i < 21; ++i) T.jframe.push_back(tp.joint_frame[21 * j + i]);
    T.jparam.push_back(tp.joint_param[2 * j]);
    T.jparam.push_back(tp.joint_param[2 * j + 1]);
  }
  T.rows_joint = row;
  for (int e = 0; e < T.nt; ++e) {
    for (int k = 0; k < 4; ++k) {
      const int b = tp.tet_body[4 * e + k];
      if (b < 0 || b >= T.nb || T.btype[b] != 0) throw NsdError(NSD_INVALID, "tet vertex must be a particle body");
      T.tbody.push_back(b);
    }
    for (int k = 0; k < 9; ++k) T.tdminv.push_back(tp.tet_dm_inv[9 * e + k]);
    T.tvol.push_back(tp.tet_volume[e]);
    for (int k = 0; k < 4; ++k) T.tmat.push_back(tp.tet_material[4 * e + k]);
  }
  // rows per tet: 3 (Neo-Hookean) or 6 (linear co-rotational, flag 2); one model per topology
  for (int e = 0; e < T.nt; ++e) {
    const int td = (static_cast<int>(T.tmat[4 * e + 3]) & 2) ? 6 : 3;
    if (e == 0) T.tdim = td;
    if (td != T.tdim)
      throw NsdError(NSD_UNSUPPORTED, "mixed Neo-Hookean and linear co-rotational meshes in one scene");
  }
  if (T.tdim == 6)
    for (int e = 0; e < T.nt; ++e) {  // K from the Lame constants: mu = 2 c1, lambda = 2 d1
      const double mu = 2.0 * T.tmat[4 * e], lam = 2.0 * T.tmat[4 * e + 1];
      double K[6][6] = {}, Ki[6][6];
      for (int i = 0; i < 3; ++i) {
        for (int j = 0; j < 3; ++j) K[i][j] = lam;
        K[i][i] = lam + 2.0 * mu;
        K[i + 3][i + 3] = mu;
      }
      inverse6_h(K, Ki);
      for (int i = 0; i < 6; ++i)
        for (int j = 0; j < 6; ++j) T.tkinv.push_back(Ki[i][j]);
    }
  T.rows_static = T.rows_joint + T.tdim * T.nt;
  // static incidence: (row, slot) per dof3 block, rows ascending
  std::vector<std::vector<int>> inc(T.nd3);
  for (int j = 0; j < T.nj; ++j) {
    int al, aa, bl, ba;
    body_blocks_h(T, T.jbody[2 * j], al, aa);
    body_blocks_h(T, T.jbody[2 * j + 1], bl, ba);
    for (int k = 0; k < nsd::joint_nrows(T.jkind[j]); ++k) {
      const bool lin = nsd::joint_row_linear(T.jkind[j], k);
      int b4[4] = {lin ? al : -1, aa, lin ? bl : -1, ba};
      if (b4[2] >= 0 && b4[2] == b4[0]) b4[2] = -1;
      if (b4[3] >= 0 && b4[3] == b4[1]) b4[3] = -1;
      const int r = T.jrow[j] + k;
      for (int s = 0; s < 4; ++s)
        if (b4[s] >= 0) inc[b4[s]].push_back(4 * r + s);
    }
  }
  for (int e = 0; e < T.nt; ++e)
    for (int i = 0; i < T.tdim; ++i) {
      const int r = T.rows_joint + T.tdim * e + i;
      for (int s = 0; s < 4; ++s) inc[T.bdof[T.tbody[4 * e + s]] / 3].push_back(4 * r + s);
    }
  T.sinc_off.assign(T.nd3 + 1, 0);
  for (int b = 0; b < T.nd3; ++b) {
    T.sinc_off[b + 1] = T.sinc_off[b] + static_cast<int>(inc[b].size());
    for (int v : inc[b]) T.sinc_ent.push_back(v);
  }
  return T;
}

// Device copy of the static topology in precision R.
template <class R> struct DevTopo {
  DBuf buf;
  nsd::Topo<R> t{};
  R* jframe = nullptr;  // the (updatable) joint frames
  void upload(const HostTopo& H) {
    Layout L;
    const size_t o_btype = L.add<int>(H.nb), o_bdof = L.add<int>(H.nb), o_bcoord = L.add<int>(H.nb),
                 o_d3b = L.add<int>(H.nd3), o_d3k = L.add<int>(H.nd3), o_jkind = L.add<int>(H.nj),
                 o_jbody = L.add<int>(2 * H.nj), o_jrow = L.add<int>(H.nj), o_tbody = L.add<int>(4 * H.nt),
                 o_soff = L.add<int>(H.nd3 + 1), o_sent = L.add<int>(H.sinc_ent.size()), o_bmass = L.add<R>(H.nb),
                 o_bin = L.add<R>(9 * H.nb), o_jparam = L.add<R>(2 * H.nj), o_jframe = L.add<R>(21 * H.nj),
                 o_tdm = L.add<R>(9 * H.nt), o_tvol = L.add<R>(H.nt), o_tmat = L.add<R>(4 * H.nt),
                 o_tkinv = L.add<R>(H.tkinv.size());
    std::vector<char> host(L.bytes, 0);
    auto put_i = [&](size_t off, const std::vector<int>& v) {
      if (!v.empty()) std::memcpy(host.data() + off, v.data(), v.size() * sizeof(int));
    };
    auto put_r = [&](size_t off, const std::vector<double>& v) {
      R* d = reinterpret_cast<R*>(host.data() + off);
      for (size_t i = 0; i < v.size(); ++i) d[i] = static_cast<R>(v[i]);
    };
    put_i(o_btype, H.btype);
    put_i(o_bdof, H.bdof);
    put_i(o_bcoord, H.bcoord);
    put_i(o_d3b, H.d3_body);
    put_i(o_d3k, H.d3_kind);
    put_i(o_jkind, H.jkind);
    put_i(o_jbody, H.jbody);
    put_i(o_jrow, H.jrow);
    put_i(o_tbody, H.tbody);
    put_i(o_soff, H.sinc_off);
    put_i(o_sent, H.sinc_ent);
    put_r(o_bmass, H.bmass);
    put_r(o_bin, H.binertia);
    put_r(o_jparam, H.jparam);
    put_r(o_jframe, H.jframe);
    put_r(o_tdm, H.tdminv);
    put_r(o_tvol, H.tvol);
    put_r(o_tmat, H.tmat);
    put_r(o_tkinv, H.tkinv);
    buf.alloc(L.bytes);
    NSD_CK(cudaMemcpy(buf.p, host.data(), L.bytes, cudaMemcpyHostToDevice));
    char* base = static_cast<char*>(buf.p);
    t.nb = H.nb;
    t.ndof = H.ndof;
    t.ncoord = H.ncoord;
    t.nd3 = H.nd3;
    t.btype = reinterpret_cast<const int*>(base + o_btype);
    t.bmass = reinterpret_cast<const R*>(base + o_bmass);
    t.binertia = reinterpret_cast<const R*>(base + o_bin);
    t.bdof = reinterpret_cast<const int*>(base + o_bdof);
    t.bcoord = reinterpret_cast<const int*>(base + o_bcoord);
    t.d3_body = reinterpret_cast<const int*>(base + o_d3b);
    t.d3_kind = reinterpret_cast<const int*>(base + o_d3k);
    t.nj = H.nj;
    t.jkind = reinterpret_cast<const int*>(base + o_jkind);
    t.jbody = reinterpret_cast<const int*>(base + o_jbody);
    t.jparam = reinterpret_cast<const R*>(base + o_jparam);
    t.jrow = reinterpret_cast<const int*>(base + o_jrow);
    t.rows_joint = H.rows_joint;
    t.nt = H.nt;
    t.tbody = reinterpret_cast<const int*>(base + o_tbody);
    t.tdminv = reinterpret_cast<const R*>(base + o_tdm);
    t.tvol = reinterpret_cast<const R*>(base + o_tvol);
    t.tmat = reinterpret_cast<const R*>(base + o_tmat);
    t.tdim = H.tdim;
    t.tkinv = reinterpret_cast<const R*>(base + o_tkinv);
    t.rows_static = H.rows_static;
    t.sinc_off = reinterpret_cast<const int*>(base + o_soff);
    t.sinc_ent = reinterpret_cast<const int*>(base + o_sent);
    // warp-cooperative J^T pull when blocks gather long incidence lists (FEM vertices sit in ~24 tets)
    t.warp_pull = H.nd3 > 0 && H.sinc_ent.size() >= 24 * static_cast<size_t>(H.nd3) ? 1 : 0;
    if (const char* e = std::getenv("NSD_WARP_PULL")) t.warp_pull = std::atoi(e);
    jframe = reinterpret_cast<R*>(base + o_jframe);
  }
};

}  // namespace

// ================================================================== handles
struct SolverBase {
  virtual ~SolverBase() = default;
  virtual int step(const nsd_step_in* in, nsd_step_out* out) = 0;
  virtual void set_cfg(const nsd_config& c) = 0;
  double last_ms = 0.0;
};

template <class R> struct Solver final : SolverBase {
  HostTopo H;
  DevTopo<R> topo;
  nsd_config cfg;
  int ccap = 0;
  WorkPlan plan;
  DBuf hotr, hoti, coldr, coldi, outbuf, gpart;
  HBuf stage_in, stage_o;
  DBuf upbuf;  // the step's inputs, one H2D copy
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  int grid_blocks = 0;
  bool use_grid = false;
  bool tets = false;
  int block_threads = 256;
  // partitioned grid PCR (nsd_part.cuh): static objects (joints, tets) split over the
  // CTAs once, contacts added per step (PartPlanH)
  std::vector<int> ps_row_begin;         // CTA p owns static rows [ps_row_begin[p], ps_row_begin[p + 1])
  std::vector<std::vector<int>> ps_blk;  // per CTA: its static rows' dof3 blocks, ascending
  std::vector<std::vector<int>> blk_ctas;  // per dof3 block: the CTAs whose static rows touch it, ascending
  DBuf partbuf;                          // shared-block partials, 3 per flat local block

  Solver(const nsd_topology& tp, const nsd_config& c, int device) : cfg(c) {
    NSD_CK(cudaSetDevice(device));
    H = preprocess(tp);
    topo.upload(H);
    tets = H.nt > 0;
    NSD_CK(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    NSD_CK(cudaEventCreate(&ev0));
    NSD_CK(cudaEventCreate(&ev1));
    ensure(16);
    const size_t work = std::max<size_t>({(size_t)H.rows_static + 48, (size_t)H.nd3, (size_t)H.nb});
    if (work <= 1536) {  // small scenes: one CTA (block barriers); larger: cooperative grid
      use_grid = false;
      block_threads = work <= 256 ? 128 : 256;  // k_single_block's launch bound
    } else {
      use_grid = true;
      int dev_sms = 0, per_sm = 0;
      NSD_CK(cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, device));
      per_sm = std::min(s64::single_grid_blocks_per_sm<R>(tets), s32::single_grid_blocks_per_sm<R>(tets));
      if (per_sm < 1) throw NsdError(NSD_CUDA_ERROR, "grid kernel cannot be resident");
      const char* bps = std::getenv("NSD_GRID_BLOCKS_PER_SM");
      grid_blocks = std::min(nsd::kGridMaxCtas, dev_sms * std::min(per_sm, bps ? std::max(1, std::atoi(bps)) : 1));
      if (const char* gc = std::getenv("NSD_GRID_CTAS")) grid_blocks = std::max(1, std::min(grid_blocks, std::atoi(gc)));
      // partials, arrival count and flag-in-data words of the grid reductions (nsd_team.cuh)
      gpart.alloc(sizeof(double) * nsd::grid_scratch_doubles(grid_blocks));
      part_static();
      int optin = 0;
      NSD_CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
      part_smem_max = optin > 8192 ? (size_t)optin - 8192 : 0;  // the team's static reduction buffer stays below
    }
  }
  size_t part_smem_max = 0;
  // partitioned grid PCR unless NSD_GRID_PART=0
  static bool part_enabled() {
    const char* e = std::getenv("NSD_GRID_PART");
    return !(e && std::atoi(e) == 0);
  }
  // Static objects (joints, then tets; all rows of an object together) over the grid's
  // CTAs in row order, balanced by rows; each CTA's blocks from the static incidence.
  void part_static() {
    const int P = grid_blocks;
    std::vector<int> starts;  // object starts in row order
    for (int j = 0; j < H.nj; ++j) starts.push_back(H.jrow[j]);
    for (int e = 0; e < H.nt; ++e) starts.push_back(H.rows_joint + H.tdim * e);
    starts.push_back(H.rows_static);
    ps_row_begin.assign(P + 1, H.rows_static);
    ps_row_begin[0] = 0;
    for (int p = 1; p < P; ++p) {
      const long target = (long)H.rows_static * p / P;
      ps_row_begin[p] = *std::lower_bound(starts.begin(), starts.end(), (int)target);
    }
    std::vector<int> owner(H.rows_static);
    for (int p = 0; p < P; ++p)
      for (int i = ps_row_begin[p]; i < ps_row_begin[p + 1]; ++i) owner[i] = p;
    ps_blk.assign(P, {});
    blk_ctas.assign(H.nd3, {});
    for (int b = 0; b < H.nd3; ++b) {
      for (int e = H.sinc_off[b]; e < H.sinc_off[b + 1]; ++e) {
        const int p = owner[H.sinc_ent[e] >> 2];
        if (ps_blk[p].empty() || ps_blk[p].back() != b) ps_blk[p].push_back(b);
        blk_ctas[b].push_back(p);
      }
      std::sort(blk_ctas[b].begin(), blk_ctas[b].end());
      blk_ctas[b].erase(std::unique(blk_ctas[b].begin(), blk_ctas[b].end()), blk_ctas[b].end());
    }
  }
  DBuf ptime;  // NSD_PHASE_TIMING: CTA 0's clock64 cycles per partitioned-PCR phase
  long n_steps = 0;
  double host_ms[4] = {0, 0, 0, 0};  // NSD_HOST_TIMING: wall ms per nsd_step host phase
  ~Solver() override {
    if (std::getenv("NSD_HOST_TIMING") && n_steps > 0)
      std::fprintf(stderr, "nsd_step host wall ms per step: stage %.4f launch %.4f download+sync+unpack %.4f (%ld steps)\n",
                   host_ms[0] / n_steps, host_ms[1] / n_steps, host_ms[2] / n_steps, n_steps);
    if (ptime.p && n_steps > 0) {  // diagnostics: cycles per phase, summed over the solver's steps
      unsigned long long h[16] = {};
      if (cudaMemcpy(h, ptime.p, sizeof(h), cudaMemcpyDeviceToHost) == cudaSuccess) {
        static const char* names[] = {"trial pass", "scatter", "reduce+gather", "row pass", "reduce"};
        std::fprintf(stderr, "nsd_step phase cycles (CTA 0, thread 0, %ld steps):", n_steps);
        for (int k = 0; k < 5; ++k) std::fprintf(stderr, " %s %llu", names[k], h[k]);
        std::fprintf(stderr, "\n");
        static const char* rn[] = {"local sums + partial store", "arrival atomic", "spin", "partial sums (+side)", "tail"};
        std::fprintf(stderr, "nsd_step grid reductions (CTA 0, thread 0, all launches' reductions and syncs):");
        for (int k = 1; k < 6; ++k) std::fprintf(stderr, " %s %llu", rn[k - 1], h[8 + k]);
        std::fprintf(stderr, "\n");
        std::vector<unsigned long long> pc(2 * (size_t)grid_blocks);
        if (cudaMemcpy(pc.data(), static_cast<unsigned long long*>(ptime.p) + 16, pc.size() * sizeof(unsigned long long),
                       cudaMemcpyDeviceToHost) == cudaSuccess) {
          for (int k = 0; k < 2; ++k) {
            unsigned long long mn = ~0ull, mx = 0, sum = 0;
            int amx = 0;
            for (int b = 0; b < grid_blocks; ++b) {
              const unsigned long long v = pc[2 * b + k];
              mn = std::min(mn, v);
              if (v > mx) { mx = v; amx = b; }
              sum += v;
            }
            std::fprintf(stderr, "nsd_step per-CTA %s cycles: min %llu mean %llu max %llu (CTA %d)\n",
                         k ? "reduction" : "compute", mn, sum / grid_blocks, mx, amx);
          }
        }
      }
    }
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    if (stream) cudaStreamDestroy(stream);
  }
  void set_cfg(const nsd_config& c) override { cfg = c; }
  void ensure(int nc) {
    if (nc <= ccap && hotr.p) return;
    ccap = std::max(nc, std::max(16, ccap * 2));
    plan.plan(H, ccap);
    hotr.alloc(plan.hot_bytes<R>());
    coldr.alloc(sizeof(R) * plan.coldR);
    coldi.alloc(sizeof(int) * plan.coldI);
  }

  int step(const nsd_step_in* in, nsd_step_out* out) override {
    if (!in || !out || !in->q || !in->u || !out->q || !out->u) throw NsdError(NSD_INVALID, "null step buffers");
    if (!(in->h > 0.0)) throw NsdError(NSD_INVALID, "integrate_coordinates: h must be positive");
    const int nc = in->n_contacts;
    if (nc < 0 || (nc > 0 && !in->contacts)) throw NsdError(NSD_INVALID, "bad contact list");
    for (int c = 0; c < nc; ++c) {
      const nsd_contact& k = in->contacts[c];
      if (k.body_a < -1 || k.body_a >= H.nb || k.body_b < -1 || k.body_b >= H.nb)
        throw NsdError(NSD_INVALID, "contact references invalid body");
    }
    ensure(nc);
    const int N = cfg.newton_iterations, ml = cfg.linear_max_iterations;
    const int nrows = H.rows_static + 3 * nc;
    Nvtx range_step("nsd_step");
    NvtxPhase phase;
    if (std::getenv("NSD_HOST_TIMING")) phase.acc = host_ms;
    phase.start("nsd_step: stage inputs (one H2D)");
    // ---- stage inputs in ONE pinned buffer and ONE H2D copy: q-, u-, f_extra, contact
    // geometry, joint frames (R part); contact bodies and the contact incidence (int
    // part). The kernel reads them in place (Work's const input pointers).
    const size_t nR = (size_t)H.ncoord + H.ndof + H.ndof + 17 * (size_t)nc + 21 * (size_t)H.nj;
    // contact incidence (contact*4 + slot), contacts ascending within a block
    std::vector<int> cnt(H.nd3 + 1, 0);
    std::vector<int> b4all(4 * (size_t)nc);
    for (int c = 0; c < nc; ++c) {
      int* b4 = &b4all[4 * c];
      body_blocks_h(H, in->contacts[c].body_a, b4[0], b4[1]);
      body_blocks_h(H, in->contacts[c].body_b, b4[2], b4[3]);
      for (int s = 0; s < 4; ++s)
        if (b4[s] >= 0) cnt[b4[s] + 1]++;
    }
    for (int b = 0; b < H.nd3; ++b) cnt[b + 1] += cnt[b];
    // ---- partitioned grid PCR plan (nsd_part.cuh): each contact goes to the least
    // loaded (fewest rows so far; ties: lowest) CTA among those whose static rows touch
    // one of its blocks (else the least loaded CTA), so its blocks stay local there
    // and ground-contact CTAs do not pile up rows; its three rows follow the CTA's
    // static rows; local blocks = static blocks + contact blocks; per dof3 block the
    // flat local-block indices of all CTAs touching it, CTA order.
    std::vector<int> p_row_off, p_rows, p_lb_off, p_lb_blk, p_gb_off, p_gb_ent;
    int p_mr = 0, p_ml = 0, p_mx = 0;
    size_t p_smem = 0;
    bool use_part = false;
    if (use_grid && cfg.linear_method == 3 && part_enabled()) {
      const int P = grid_blocks;
      std::vector<int> cstart(P + 1, 0), cown(nc), clist(nc), load(P);
      for (int p = 0; p < P; ++p) load[p] = ps_row_begin[p + 1] - ps_row_begin[p];
      for (int c = 0; c < nc; ++c) {
        const int* b4 = &b4all[4 * c];
        int o = -1;
        for (int s = 0; s < 4; ++s)
          if (b4[s] >= 0)
            for (int p : blk_ctas[b4[s]])
              if (o < 0 || load[p] < load[o] || (load[p] == load[o] && p < o)) o = p;
        if (o < 0)
          o = static_cast<int>(std::min_element(load.begin(), load.end()) - load.begin());
        cown[c] = o;
        load[o] += 3;
        cstart[cown[c] + 1]++;
      }
      for (int p = 0; p < P; ++p) cstart[p + 1] += cstart[p];
      {
        std::vector<int> fp(cstart.begin(), cstart.end() - 1);
        for (int c = 0; c < nc; ++c) clist[fp[cown[c]]++] = c;
      }
      p_row_off.assign(P + 1, 0);
      p_rows.reserve(nrows);
      p_lb_off.assign(P + 1, 0);
      std::vector<int> extra, merged;
      for (int p = 0; p < P; ++p) {
        for (int i = ps_row_begin[p]; i < ps_row_begin[p + 1]; ++i) p_rows.push_back(i);
        extra.clear();
        for (int k = cstart[p]; k < cstart[p + 1]; ++k) {
          const int c = clist[k];
          p_rows.push_back(H.rows_static + c);
          p_rows.push_back(H.rows_static + nc + 2 * c);
          p_rows.push_back(H.rows_static + nc + 2 * c + 1);
          for (int s = 0; s < 4; ++s)
            if (b4all[4 * c + s] >= 0) extra.push_back(b4all[4 * c + s]);
        }
        p_row_off[p + 1] = (int)p_rows.size();
        p_mr = std::max(p_mr, p_row_off[p + 1] - p_row_off[p]);
        if (extra.empty()) {
          p_lb_blk.insert(p_lb_blk.end(), ps_blk[p].begin(), ps_blk[p].end());
        } else {
          std::sort(extra.begin(), extra.end());
          extra.erase(std::unique(extra.begin(), extra.end()), extra.end());
          merged.clear();
          std::set_union(ps_blk[p].begin(), ps_blk[p].end(), extra.begin(), extra.end(), std::back_inserter(merged));
          p_lb_blk.insert(p_lb_blk.end(), merged.begin(), merged.end());
        }
        p_lb_off[p + 1] = (int)p_lb_blk.size();
        p_ml = std::max(p_ml, p_lb_off[p + 1] - p_lb_off[p]);
      }
      const int nlb = (int)p_lb_blk.size();
      p_gb_off.assign(H.nd3 + 1, 0);
      for (int f = 0; f < nlb; ++f) p_gb_off[p_lb_blk[f] + 1]++;
      for (int b = 0; b < H.nd3; ++b) p_gb_off[b + 1] += p_gb_off[b];
      p_gb_ent.resize(std::max(nlb, 1));
      {
        std::vector<int> fp(p_gb_off.begin(), p_gb_off.end() - 1);
        for (int f = 0; f < nlb; ++f) p_gb_ent[fp[p_lb_blk[f]]++] = f;  // f ascending = CTA order
      }
      for (int p = 0; p < P; ++p) {
        int x = 0;
        for (int f = p_lb_off[p]; f < p_lb_off[p + 1]; ++f) x += p_gb_off[p_lb_blk[f] + 1] - p_gb_off[p_lb_blk[f]];
        p_mx = std::max(p_mx, x);
      }
      p_smem = nsd::part_smem<R>(std::max(p_mr, 1), std::max(p_ml, 1), std::max(p_mx, 1)).bytes;
      use_part = (int)p_rows.size() == nrows && p_smem <= part_smem_max;
      if (use_part) partbuf.alloc(sizeof(R) * 3 * (size_t)std::max(nlb, 1));
    }
    const size_t n_part = use_part ? p_row_off.size() + p_rows.size() + p_lb_off.size() + p_lb_blk.size() +
                                         p_gb_off.size() + p_gb_ent.size()
                                   : 0;
    const size_t nI = 2 * (size_t)nc + (H.nd3 + 1) + 4 * (size_t)nc + n_part;
    Layout U;
    const size_t u_r = U.add<R>(nR), u_i = U.add<int>(nI);
    stage_in.alloc(U.bytes);
    upbuf.alloc(U.bytes);
    R* sr = reinterpret_cast<R*>(static_cast<char*>(stage_in.p) + u_r);
    int* si = reinterpret_cast<int*>(static_cast<char*>(stage_in.p) + u_i);
    size_t o = 0;
    for (int i = 0; i < H.ncoord; ++i) sr[o++] = R(in->q[i]);
    for (int i = 0; i < H.ndof; ++i) sr[o++] = R(in->u[i]);
    for (int i = 0; i < H.ndof; ++i) sr[o++] = in->f_extra ? R(in->f_extra[i]) : R(0);
    for (int c = 0; c < nc; ++c) {
      const nsd_contact& k = in->contacts[c];
      for (int i = 0; i < 3; ++i) sr[o + i] = R(k.local_a[i]);
      for (int i = 0; i < 3; ++i) sr[o + 3 + i] = R(k.local_b[i]);
      for (int i = 0; i < 3; ++i) sr[o + 6 + i] = R(k.normal[i]);
      for (int i = 0; i < 3; ++i) sr[o + 9 + i] = R(k.d1[i]);
      for (int i = 0; i < 3; ++i) sr[o + 12 + i] = R(k.d2[i]);
      sr[o + 15] = R(k.thickness);
      sr[o + 16] = R(k.mu);
      o += 17;
    }
    const double* jf = in->joint_frame ? in->joint_frame : H.jframe.data();
    for (int i = 0; i < 21 * H.nj; ++i) sr[o++] = R(jf[i]);
    for (int c = 0; c < nc; ++c) {
      si[2 * c] = in->contacts[c].body_a;
      si[2 * c + 1] = in->contacts[c].body_b;
    }
    int* soff = si + 2 * nc;
    int* sent = soff + H.nd3 + 1;
    for (int b = 0; b <= H.nd3; ++b) soff[b] = cnt[b];
    {
      std::vector<int> fillp(cnt.begin(), cnt.end() - 1);
      for (int c = 0; c < nc; ++c)
        for (int s = 0; s < 4; ++s) {
          const int b = b4all[4 * c + s];
          if (b >= 0) sent[fillp[b]++] = 4 * c + s;
        }
    }
    {
      int* pi = sent + 4 * (size_t)nc;
      for (const std::vector<int>* v : {&p_row_off, &p_rows, &p_lb_off, &p_lb_blk, &p_gb_off, &p_gb_ent})
        if (use_part) {
          std::memcpy(pi, v->data(), v->size() * sizeof(int));
          pi += v->size();
        }
    }
    R* hr = hotr.as<R>();
    int* hi = plan.hot_ints(hr);
    R* cr = coldr.as<R>();
    int* ci = coldi.as<int>();
    NSD_CK(cudaMemcpyAsync(upbuf.p, stage_in.p, U.bytes, cudaMemcpyHostToDevice, stream));
    const R* dr = reinterpret_cast<const R*>(upbuf.as<char>() + u_r);
    const int* di = reinterpret_cast<const int*>(upbuf.as<char>() + u_i);
    // ---- outputs
    Layout L;
    const int dec_stride = nc + H.nt + H.ndof + 1;
    const size_t o_it = L.add<nsd::IterOut>(N), o_hist = L.add<double>((size_t)N * (ml + 1)),
                 o_hl = L.add<int>(N), o_tel = L.add<double>(6 * (size_t)nc), o_fin = L.add<double>(8),
                 o_dec = L.add<unsigned char>((size_t)N * dec_stride), o_q = L.add<R>(H.ncoord),
                 o_u = L.add<R>(H.ndof), o_lam = L.add<R>(nrows);
    outbuf.alloc(L.bytes);
    char* ob = outbuf.as<char>();
    NSD_CK(cudaMemsetAsync(ob, 0, L.bytes, stream));
    nsd::StepOut so{};
    so.iters = reinterpret_cast<nsd::IterOut*>(ob + o_it);
    so.hist = reinterpret_cast<double*>(ob + o_hist);
    so.hist_len = reinterpret_cast<int*>(ob + o_hl);
    so.tel = reinterpret_cast<double*>(ob + o_tel);
    so.fin = reinterpret_cast<double*>(ob + o_fin);
    so.dec = out->decisions ? reinterpret_cast<unsigned char*>(ob + o_dec) : nullptr;
    so.dec_stride = dec_stride;
    if (std::getenv("NSD_PHASE_TIMING") && use_grid) {
      if (!ptime.p) {
        ptime.alloc(sizeof(unsigned long long) * (16 + 2 * (size_t)grid_blocks));
        NSD_CK(cudaMemset(ptime.p, 0, sizeof(unsigned long long) * (16 + 2 * (size_t)grid_blocks)));
      }
      so.ptime = ptime.as<unsigned long long>();
    }
    ++n_steps;
    nsd::Work<R> W = plan.bind<R>(hr, hi, cr, ci);
    // inputs in place in the upload buffer; q, u, lambda in the output buffer (one D2H)
    W.q0 = dr;
    W.u0 = dr + H.ncoord;
    W.f_extra = in->f_extra ? dr + H.ncoord + H.ndof : nullptr;
    W.cgeo = dr + H.ncoord + 2 * H.ndof;
    W.jframe = dr + H.ncoord + 2 * H.ndof + 17 * (size_t)nc;
    W.cbody = di;
    W.cinc_off = di + 2 * nc;
    W.cinc_ent = di + 2 * nc + H.nd3 + 1;
    W.part_row_off = W.part_rows = W.part_lb_off = W.part_lb_blk = W.part_gb_off = W.part_gb_ent = nullptr;
    W.part_partial = nullptr;
    W.part_mr = W.part_ml = W.part_mx = 0;
    if (use_part) {
      const int* pi = di + 2 * nc + (H.nd3 + 1) + 4 * (size_t)nc;
      W.part_row_off = pi;
      W.part_rows = (pi += p_row_off.size());
      W.part_lb_off = (pi += p_rows.size());
      W.part_lb_blk = (pi += p_lb_off.size());
      W.part_gb_off = (pi += p_lb_blk.size());
      W.part_gb_ent = (pi += p_gb_off.size());
      W.part_partial = partbuf.p;
      W.part_mr = std::max(p_mr, 1);
      W.part_ml = std::max(p_ml, 1);
      W.part_mx = std::max(p_mx, 1);
    }
    W.q = reinterpret_cast<R*>(ob + o_q);
    W.u = reinterpret_cast<R*>(ob + o_u);
    W.lam = reinterpret_cast<R*>(ob + o_lam);
    W.h = R(in->h);
    for (int k = 0; k < 3; ++k) W.grav[k] = R(in->gravity[k]);
    W.nc = nc;
    W.nrows = nrows;
    W.normal_begin = H.rows_static;
    W.friction_begin = H.rows_static + nc;
    nsd::Cfg kc = to_cfg(cfg);
    phase.start(use_grid ? "nsd_step: newton_step (persistent cooperative grid)" : "nsd_step: newton_step (one CTA)");
    NSD_CK(cudaEventRecord(ev0, stream));
    if (!use_grid) {
      // fp32 mode: the kernels that store the J/C coefficients as float (nsd_k_single32.cu)
      NSD_CK(cfg.precision == NSD_FP32 ? s32::launch_single_block<R>(tets, block_threads, stream, topo.t, W, kc, so)
                                       : s64::launch_single_block<R>(tets, block_threads, stream, topo.t, W, kc, so));
    } else {
      double* gp = gpart.as<double>();
      NSD_CK(cudaMemsetAsync(gp + nsd::grid_scratch_reset_off(grid_blocks), 0,
                             sizeof(double) * (nsd::grid_scratch_doubles(grid_blocks) - nsd::grid_scratch_reset_off(grid_blocks)),
                             stream));  // arrival count and flag words: epochs restart every launch
      // register-resident PCR rows when every thread owns <= 2 rows (NSD_GRID_REGS=0 disables)
      const bool regs = cfg.linear_method == 3 && nrows <= 2 * grid_blocks * kGridThreads && !(std::getenv("NSD_GRID_REGS") &&
                                                                       std::atoi(std::getenv("NSD_GRID_REGS")) == 0);
      const int mode = use_part ? -1 : (regs ? 2 : 0);
      NSD_CK(cfg.precision == NSD_FP32
                 ? s32::launch_single_grid<R>(tets, mode, p_smem, grid_blocks, stream, topo.t, W, kc, so, gp)
                 : s64::launch_single_grid<R>(tets, mode, p_smem, grid_blocks, stream, topo.t, W, kc, so, gp));
    }
    NSD_CK(cudaEventRecord(ev1, stream));
    phase.start("nsd_step: download (one D2H) + unpack");
    // ---- download: one D2H of the output buffer (reports, q, u, lambda)
    stage_o.alloc(L.bytes);
    char* ho = static_cast<char*>(stage_o.p);
    NSD_CK(cudaMemcpyAsync(ho, ob, L.bytes, cudaMemcpyDeviceToHost, stream));
    const R* hq = reinterpret_cast<const R*>(ho + o_q);
    const R* hu = reinterpret_cast<const R*>(ho + o_u);
    const R* hl = reinterpret_cast<const R*>(ho + o_lam);
    NSD_CK(cudaStreamSynchronize(stream));
    float ms = 0.f;
    NSD_CK(cudaEventElapsedTime(&ms, ev0, ev1));
    last_ms = ms;
    const double* fin = reinterpret_cast<const double*>(ho + o_fin);
    const nsd::IterOut* its = reinterpret_cast<const nsd::IterOut*>(ho + o_it);
    const int nit = static_cast<int>(fin[7]);
    const bool aborted = fin[5] != 0.0;
    for (int i = 0; i < H.ncoord; ++i) out->q[i] = double(hq[i]);
    for (int i = 0; i < H.ndof; ++i) out->u[i] = double(hu[i]);
    if (out->lambda)
      for (int i = 0; i < nrows; ++i) out->lambda[i] = double(hl[i]);
    if (out->iters)
      for (int i = 0; i < nit; ++i) {
        nsd_iter_stats& s = out->iters[i];
        s.residual_inf = its[i].residual_inf;
        s.merit_l2 = its[i].merit_l2;
        s.comp_error_max = its[i].comp_error_max;
        s.cone_violation_max = its[i].cone_violation_max;
        s.step_size = its[i].step_size;
        s.linear_residual = its[i].linear_residual;
        s.linear_iterations = its[i].linear_iterations;
        s.linear_breakdown = its[i].linear_breakdown;
      }
    if (out->linear_history) {
      const double* hh = reinterpret_cast<const double*>(ho + o_hist);
      std::memcpy(out->linear_history, hh, sizeof(double) * (size_t)N * (ml + 1));
    }
    if (out->linear_history_len) std::memcpy(out->linear_history_len, ho + o_hl, sizeof(int) * N);
    if (out->decisions) std::memcpy(out->decisions, ho + o_dec, (size_t)N * dec_stride);
    if (out->contact_telemetry && nc && !aborted)
      std::memcpy(out->contact_telemetry, ho + o_tel, sizeof(double) * 6 * nc);
    if (out->contacts && !aborted) {
      const int nb0 = H.rows_static, fb0 = H.rows_static + nc;
      for (int c = 0; c < nc; ++c) {
        if (out->contacts != in->contacts) out->contacts[c] = in->contacts[c];
        out->contacts[c].lambda_n = double(hl[nb0 + c]);
        out->contacts[c].lambda_f[0] = double(hl[fb0 + 2 * c]);
        out->contacts[c].lambda_f[1] = double(hl[fb0 + 2 * c + 1]);
      }
    }
    out->n_iterations = nit;
    out->n_rows = nrows;
    out->final_residual_inf = fin[0];
    out->final_comp_error = fin[1];
    out->final_cone_violation = fin[2];
    out->min_gap = fin[3];
    out->min_diag_shift = fin[4];
    out->aborted = aborted ? 1 : 0;
    out->converged = fin[6] != 0.0 ? 1 : 0;
    return aborted ? NSD_ABORTED : NSD_OK;
  }
};

struct BatchBase {
  virtual ~BatchBase() = default;
  virtual void set_state(const double* q, const double* u) = 0;
  virtual void get_state(double* q, double* u) = 0;
  virtual void step(const void* torque, int on_device, int dtype, double h, const double* g, void* q_out = nullptr,
                    void* u_out = nullptr) = 0;
  virtual void results(int* nc, int* ab, double* fres, nsd_iter_stats* its) = 0;
  virtual void contacts(int env, nsd_contact* out, int* n) = 0;
  virtual void device_state(void** q, void** u, int* dtype) = 0;
  virtual void copy_state_async(void* q, void* u) = 0;
  virtual void counters(unsigned long long* out) = 0;
  virtual void set_profile(int on) = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = true;
  int info[6] = {0, 0, 0, 0, 0, 0};
};

template <class R> struct Batch final : BatchBase {
  HostTopo H;
  DevTopo<R> topo;
  nsd_config cfg;
  int n_env, maxc, ns, npairs;
  WorkPlan plan;
  DBuf hotg, coldr, coldi, shapes, pairs, cand, paircnt, ncout, ovf, fin, iters, qs, us, torque, jbinc, jblk;
  DBuf abany, ctr, wjinc, wlam, wptime, porder;  // sticky abort flags; counters; k_batch_warp's joint incidence (both sides)
  bool warp_path = false;  // k_batch_warp for rigid scenes (narrow-phase launch + warp solver + large-env launch)
  nsd::wp::Plan wplan{};
  int warp_epb = 2;        // environments (warps) per block of k_batch_warp (64 threads, 7 blocks/SM)
  int warp_max_obj = 32;   // NSD_WARP_MAX_OBJ (tests) routes smaller envs to the object solver too
  int collide_cap = 64;    // k_batch_collide's per-env candidate list (>= max_contacts)
  size_t collide_smem = 0;
  DBuf wsetup;             // rigid path: per env u~, I_w, I_w^-1
  size_t warp_smem = 0;
  long env_steps = 0;
  bool profile = false;     // bit 0 of nsd_batch_profile: in-kernel cycle counters
  bool time_launches = false;  // bit 1: CUDA events around each launch of the step
  std::vector<cudaEvent_t> evpool;  // 4 per timed step: before narrow phase, after it, after warp, after large
  size_t ev_used = 0;
  int jbinc_n = 0;
  HBuf stage;
  double margin, mu_default;
  int team_threads = 32;  // 32: warp per env; >32: CTA per env
  int envs_per_block = 4;
  bool hot_in_smem = false;  // measured: L1-cached global beats smem-limited residency
  size_t smem_bytes = 0;
  int row_pool = 0;  // per-env shared-memory row region (elements), see the constructor
  DBuf ptime;        // NSD_PHASE_TIMING counters
  std::vector<nsd::ShapeD<R>> hshapes;

  bool mixed = false;  // precision fp32 on the warp path: fp64 state, fp32 PCR operator
  Batch(const nsd_topology& tp, int n_shapes, const nsd_shape* sh, double mg, double mud, const nsd_config& c,
        int nenv, int mc, int device, bool mixed_precision = false)
      : cfg(c), n_env(nenv), maxc(mc), ns(n_shapes), margin(mg), mu_default(mud), mixed(mixed_precision) {
    NSD_CK(cudaSetDevice(device));
    if (nenv < 1 || mc < 1 || n_shapes < 0) throw NsdError(NSD_INVALID, "bad batch sizes");
    H = preprocess(tp);
    if (H.nt > 0) throw NsdError(NSD_UNSUPPORTED, "batched path: tetrahedral meshes run through nsd_step");
    topo.upload(H);
    for (int i = 0; i < ns; ++i) {
      nsd::ShapeD<R> s{};
      s.body = sh[i].body;
      s.kind = sh[i].kind;
      if (s.body >= H.nb || s.body < -1 || s.kind < 0 || s.kind > 2) throw NsdError(NSD_INVALID, "bad shape");
      for (int k = 0; k < 3; ++k) {
        s.n[k] = R(sh[i].normal[k]);
        s.he[k] = R(sh[i].half_extents[k]);
      }
      s.offset = R(sh[i].offset);
      s.radius = R(sh[i].radius);
      s.thick = R(sh[i].thickness);
      s.mu = R(sh[i].mu);
      hshapes.push_back(s);
    }
    std::vector<int2> hp;
    for (int i = 0; i < ns; ++i)
      for (int j = i + 1; j < ns; ++j) hp.push_back(make_int2(i, j));
    npairs = static_cast<int>(hp.size());
    {  // the warp narrow phase runs the pairs grouped by kind pair, most expensive first
      std::vector<int> order(npairs);
      for (int k = 0; k < npairs; ++k) order[k] = k;
      auto cls = [&](int k) {
        const int a = sh[hp[k].x].kind, b = sh[hp[k].y].kind;
        const int lo = std::min(a, b), hi = std::max(a, b);  // 0 half-space, 1 sphere, 2 box
        return lo == 2 ? 0 : (hi == 2 && lo == 1 ? 1 : (hi == 2 ? 2 : (lo == 1 ? 3 : 4)));
      };
      std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return cls(x) < cls(y); });
      porder.alloc(sizeof(int) * std::max(npairs, 1));
      if (npairs) NSD_CK(cudaMemcpy(porder.p, order.data(), sizeof(int) * npairs, cudaMemcpyHostToDevice));
    }
    shapes.alloc(sizeof(nsd::ShapeD<R>) * std::max(ns, 1));
    pairs.alloc(sizeof(int2) * std::max(npairs, 1));
    if (ns) NSD_CK(cudaMemcpy(shapes.p, hshapes.data(), sizeof(nsd::ShapeD<R>) * ns, cudaMemcpyHostToDevice));
    if (npairs) NSD_CK(cudaMemcpy(pairs.p, hp.data(), sizeof(int2) * npairs, cudaMemcpyHostToDevice));
    plan.plan(H, maxc);
    if (cfg.line_search) throw NsdError(NSD_UNSUPPORTED, "batched path: line search runs through nsd_step");
    if (cfg.linear_method != 3) throw NsdError(NSD_UNSUPPORTED, "batched path: PCR only (Jacobi/PCG run through nsd_step)");
    {  // static joint incidence per body for the warp solver: joint*2 + side (merged same-body -> side 0)
      std::vector<std::vector<int>> per(H.nb);
      for (int j = 0; j < H.nj; ++j) {
        const int a = H.jbody[2 * j], b = H.jbody[2 * j + 1];
        if (a >= 0) per[a].push_back(2 * j);
        if (b >= 0 && b != a) per[b].push_back(2 * j + 1);
      }
      std::vector<int> flat(H.nb + 1, 0);
      for (int b = 0; b < H.nb; ++b) flat[b + 1] = flat[b] + static_cast<int>(per[b].size());
      for (int b = 0; b < H.nb; ++b) flat.insert(flat.end(), per[b].begin(), per[b].end());
      jbinc_n = static_cast<int>(flat.size());
      jbinc.alloc(sizeof(int) * flat.size());
      NSD_CK(cudaMemcpy(jbinc.p, flat.data(), sizeof(int) * flat.size(), cudaMemcpyHostToDevice));
      // static dof3 blocks per joint (body_blocks of both sides), one int4 each
      std::vector<int4> jb(std::max(H.nj, 1));
      auto blocks = [&](int b, int& lin, int& ang) {
        lin = b < 0 ? -1 : H.bdof[b] / 3;
        ang = b >= 0 && H.btype[b] == 1 ? lin + 1 : -1;
      };
      for (int j = 0; j < H.nj; ++j) {
        int al, aa, bl, ba;
        blocks(H.jbody[2 * j], al, aa);
        blocks(H.jbody[2 * j + 1], bl, ba);
        jb[j] = make_int4(al, aa, bl, ba);
      }
      jblk.alloc(sizeof(int4) * jb.size());
      NSD_CK(cudaMemcpy(jblk.p, jb.data(), sizeof(int4) * jb.size(), cudaMemcpyHostToDevice));
    }
    // Team shape: TPE lanes per env (4/8/16/32, sub-warp object solver) or a CTA per
    // env (64/128/256, generic engine). Default 16 lanes (2 envs per warp): with the
    // register cap above, 4096 envs run in one wave at 14 warps/SM (measured best,
    // DESIGN.md §6).
    const char* env_team = std::getenv("NSD_BATCH_TEAM");
    team_threads = 16;
    if (env_team) team_threads = std::atoi(env_team);
    if (team_threads != 4 && team_threads != 8 && team_threads != 16 && team_threads != 32 && team_threads != 64 &&
        team_threads != 128 && team_threads != 256)
      throw NsdError(NSD_INVALID, "NSD_BATCH_TEAM must be 4, 8, 16, 32, 64, 128 or 256");
    const bool sub = team_threads <= 32;
    envs_per_block = sub ? 32 / team_threads : 1;  // one warp per block by default
    const char* env_epb = std::getenv("NSD_ENVS_PER_BLOCK");
    if (env_epb && sub) envs_per_block = std::max(1, std::min(128 / team_threads, std::atoi(env_epb)));
    const char* env_smem = std::getenv("NSD_HOT_SMEM");
    if (env_smem) hot_in_smem = std::atoi(env_smem) != 0;
    const size_t hb = plan.hot_bytes<R>();
    int max_optin = 0;
    NSD_CK(cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
    smem_bytes = hb * envs_per_block;
    if (smem_bytes > (size_t)max_optin) hot_in_smem = false;
    if (!hot_in_smem) {
      smem_bytes = 0;
      hotg.alloc(hb * n_env);
      int carve = 0;  // no shared memory: the unified L1/smem array goes to L1
      if (sub) {
        // Row pool: a per-env shared-memory region for the write-heavy PCR state
        // (global stores are write-through to L2; measured 4.9 GB of L2 writes per
        // fp64 launch without it). Sized so that every block of the launch is
        // resident at once; envs whose contact count does not fit use global.
        int sms = 0, smem_sm = 0, reserved = 0;
        NSD_CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
        NSD_CK(cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, device));
        NSD_CK(cudaDeviceGetAttribute(&reserved, cudaDevAttrReservedSharedMemoryPerBlock, device));
        const int nblk = (n_env + envs_per_block - 1) / envs_per_block;
        const int bps = std::max(1, std::min(32, (nblk + sms - 1) / sms));
        // shared memory is allocated in 128-byte units: an allowance that ignores the
        // rounding can lose a block per SM (a second wave)
        const long unit = 128;
        const long budget = std::min<long>(max_optin, (smem_sm / bps - reserved) / unit * unit);
        const int full = row_pool_elems<R>(H.rows_static, H.nj, H.ndof, maxc);
        int region = static_cast<int>(budget / envs_per_block / static_cast<long>(sizeof(R))) & ~3;
        region = std::min(region, full);
        // Region contact capacity (envs with more contacts use global memory): the rest
        // of the unified L1/shared array stays L1 for the read-mostly data. Measured
        // (C5, 4096 envs): fp32 best at 20-26 contacts (3.62 M env-steps/s
        // vs 3.14 M sized for all 48 = 96% carveout); fp64 best filling the budget
        // (~17 contacts). NSD_POOL_NC overrides.
        int pool_nc = sizeof(R) == 4 ? 24 : maxc;
        if (const char* e = std::getenv("NSD_POOL_NC")) pool_nc = std::max(1, std::atoi(e));
        region = std::min(region, row_pool_elems<R>(H.rows_static, H.nj, H.ndof, std::min(pool_nc, maxc)));
        const char* env_rp = std::getenv("NSD_ROW_SMEM");
        if (env_rp && std::atoi(env_rp) == 0) region = 0;
        if (region < row_pool_elems<R>(H.rows_static, H.nj, H.ndof, 1)) region = 0;
        row_pool = region;
        smem_bytes = static_cast<size_t>(region) * envs_per_block * sizeof(R);
        if (smem_bytes) {
          // the limit is a per-function attribute shared by every Batch: set it to the
          // device maximum (a permission, not an allocation) so handles cannot shrink it
          // under one another
          const int sb = static_cast<int>(smem_bytes);
          NSD_CK(batch_sub_attrs<R>(max_optin, -1));
          carve = static_cast<int>(std::min<long>(100, (100L * bps * (sb + reserved) + smem_sm - 1) / smem_sm));
        }
        if (std::getenv("NSD_VERBOSE"))
          std::fprintf(stderr, "nsd batch: %d envs, %d blocks/SM, row pool %d elems/env (full %d, %zu B/block), carveout %d\n",
                       n_env, bps, region, full, smem_bytes, carve);
      }
      if (const char* e = std::getenv("NSD_L1_CARVEOUT")) carve = std::atoi(e);
      NSD_CK(batch_sub_attrs<R>(-1, carve));
    } else {
      NSD_CK(batch_sub_attrs<R>(max_optin, -1));
      NSD_CK(batch_block_attrs<R>(max_optin));
    }
    coldr.alloc(sizeof(R) * plan.coldR * n_env);
    coldi.alloc(sizeof(int) * plan.coldI * n_env);
    NSD_CK(cudaMemset(coldr.p, 0, sizeof(R) * plan.coldR * n_env));
    NSD_CK(cudaMemset(coldi.p, 0, sizeof(int) * plan.coldI * n_env));
    cand.alloc(sizeof(nsd::CandD<R>) * (size_t)std::max(npairs, 1) * 4 * n_env);
    paircnt.alloc(sizeof(int) * (size_t)std::max(npairs, 1) * n_env);
    ncout.alloc(sizeof(int) * n_env);
    ovf.alloc(sizeof(int) * n_env);
    fin.alloc(sizeof(double) * 8 * n_env);
    iters.alloc(sizeof(nsd::IterOut) * (size_t)std::max(cfg.newton_iterations, 1) * n_env);
    qs.alloc(sizeof(R) * (size_t)H.ncoord * n_env);
    us.alloc(sizeof(R) * (size_t)H.ndof * n_env);
    torque.alloc(sizeof(double) * (size_t)std::max(H.nj, 1) * n_env);
    NSD_CK(cudaMemset(ncout.p, 0, sizeof(int) * n_env));
    NSD_CK(cudaMemset(ovf.p, 0, sizeof(int) * n_env));
    NSD_CK(cudaMemset(fin.p, 0, sizeof(double) * 8 * n_env));
    NSD_CK(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    info[0] = n_env;
    info[1] = H.ncoord;
    info[2] = H.ndof;
    info[3] = H.nj;
    info[4] = H.rows_static + 3 * maxc;
    info[5] = team_threads;
    if (std::getenv("NSD_PHASE_TIMING")) {
      ptime.alloc(sizeof(unsigned long long) * 16);
      NSD_CK(cudaMemset(ptime.p, 0, sizeof(unsigned long long) * 16));
    }
    abany.alloc(sizeof(int) * n_env);
    NSD_CK(cudaMemset(abany.p, 0, sizeof(int) * n_env));
    ctr.alloc(sizeof(unsigned long long) * 4);
    NSD_CK(cudaMemset(ctr.p, 0, sizeof(unsigned long long) * 4));
    // Warp-per-env solver (nsd_warp.cuh): rigid bodies only, <= 32 bodies and joints,
    // the default team shape and slabs in global memory (NSD_BATCH_FAST=0 disables).
    bool all_rigid = H.nb > 0;
    for (int b = 0; b < H.nb; ++b) all_rigid = all_rigid && H.btype[b] == 1;
    const char* fe = std::getenv("NSD_BATCH_FAST");
    warp_path = all_rigid && H.nb <= 32 && H.nj <= 32 && team_threads == 16 && !env_team && !hot_in_smem &&
                !(fe && std::atoi(fe) == 0);
    if (warp_path) {
      std::vector<std::vector<int>> per(H.nb);
      for (int j = 0; j < H.nj; ++j) {
        const int a = H.jbody[2 * j], b = H.jbody[2 * j + 1];
        if (a >= 0) per[a].push_back(2 * j);
        if (b >= 0) per[b].push_back(2 * j + 1);
      }
      std::vector<int> flat(H.nb + 1, 0);
      for (int b = 0; b < H.nb; ++b) flat[b + 1] = flat[b] + static_cast<int>(per[b].size());
      for (int b = 0; b < H.nb; ++b) flat.insert(flat.end(), per[b].begin(), per[b].end());
      wjinc.alloc(sizeof(int) * flat.size());
      NSD_CK(cudaMemcpy(wjinc.p, flat.data(), sizeof(int) * flat.size(), cudaMemcpyHostToDevice));
      wplan = mixed ? nsd::wp::Plan::make<R, float>(H.nb) : nsd::wp::Plan::make<R, R>(H.nb);
      wlam.alloc(sizeof(R) * nsd::wp::kRows * 32 * (size_t)n_env);
      if (std::getenv("NSD_PHASE_TIMING")) {
        wptime.alloc(sizeof(unsigned long long) * nsd::wp::kWPhases);
        NSD_CK(cudaMemset(wptime.p, 0, sizeof(unsigned long long) * nsd::wp::kWPhases));
      }
      if (const char* e = std::getenv("NSD_WARP_EPB")) warp_epb = std::max(1, std::min(8, std::atoi(e)));
      if (const char* e = std::getenv("NSD_WARP_MAX_OBJ")) warp_max_obj = std::max(0, std::min(32, std::atoi(e)));
      collide_cap = std::max(64, maxc);
      const int nview = (H.ncoord + H.ndof + 9 * H.nb + 1) & ~1;
      collide_smem = 4 * (sizeof(R) * nview + sizeof(int4) * collide_cap);
      wsetup.alloc(sizeof(R) * (size_t)(H.ndof + 12 * H.nd3) * n_env);
      warp_smem = static_cast<size_t>(wplan.bytes) * warp_epb;
      int per_sm = 0;
      NSD_CK(batch_warp_setup<R>(mixed, max_optin, 32 * warp_epb, warp_smem, &per_sm));
      if (per_sm < 1) warp_path = false;
      if (std::getenv("NSD_VERBOSE"))
        std::fprintf(stderr, "nsd batch warp path: %d B/env, %d envs/block, %d blocks/SM\n", wplan.bytes, warp_epb,
                     per_sm);
    }
  }
  ~Batch() override {
    if (ptime.p) {  // diagnostics: cycles per phase summed over envs (team leaders)
      unsigned long long h[16];
      cudaStreamSynchronize(stream);
      cudaMemcpy(h, ptime.p, sizeof(h), cudaMemcpyDeviceToHost);
      static const char* names[16] = {"torque+setup+collide", "assemble", "momentum", "b/precond+tail",
                                      "pcr A (p,ap,den)", "pcr B (trial norms)", "pcr commit", "pcr stage J^T z",
                                      "pcr bodies H^-1", "pcr J w (+za)", "du/NaN", "update+integrate",
                                      "final assemble", "incidence+rowblk", "", ""};
      unsigned long long tot = 0, solver = 0;
      for (int k = 0; k < 13; ++k) tot += h[k];
      for (int k = 1; k < 13; ++k) solver += h[k];
      h[13] = h[13] > solver ? h[13] - solver : 0;  // batch_env's clock spans incidence + the solver
      tot += h[13];
      std::fprintf(stderr, "nsd phase timing (%d envs, %s):\n", n_env, sizeof(R) == 8 ? "fp64" : "fp32");
      for (int k = 0; k < 14; ++k)
        std::fprintf(stderr, "  %-24s %6.2f%%  %.3g cycles/env\n", names[k], tot ? 100.0 * h[k] / tot : 0.0,
                     double(h[k]) / n_env);
      std::fprintf(stderr, "  env time: max %.3g cycles (one step), mean %.3g cycles per env-step\n", double(h[14]),
                   double(h[15]) / std::max(1.0, double(launches) * n_env));
    }
    if (wptime.p) {  // diagnostics: the warp solver's lane-0 cycles per phase, summed over envs
      unsigned long long h[nsd::wp::kWPhases];
      cudaStreamSynchronize(stream);
      cudaMemcpy(h, wptime.p, sizeof(h), cudaMemcpyDeviceToHost);
      static const char* names[nsd::wp::kWPhases] = {
          "setup+incidence", "assemble", "momentum (g, w)", "rhs/precond + PCR tail", "PCR A z setup",
          "PCR A (p, ap, den)", "PCR trial + stage J^T z'", "PCR accept", "PCR bodies H^-1 J^T",
          "PCR J w (az, zaz)", "du / NaN check", "update + integrate", "final assemble", "write-back"};
      unsigned long long tot = 0;
      for (int k = 0; k < nsd::wp::kWPhases; ++k) tot += h[k];
      std::fprintf(stderr, "nsd warp-solver phase timing (%d envs, %s):\n", n_env, sizeof(R) == 8 ? "fp64" : "fp32");
      for (int k = 0; k < nsd::wp::kWPhases; ++k)
        std::fprintf(stderr, "  %-28s %6.2f%%  %.4g cycles/env-step\n", names[k], tot ? 100.0 * h[k] / tot : 0.0,
                     double(h[k]) / std::max(1.0, double(launches) * n_env));
    }
    for (cudaEvent_t e : evpool) cudaEventDestroy(e);
    if (stream && own_stream) cudaStreamDestroy(stream);
  }
  void set_state(const double* q, const double* u) override {
    const size_t nq = (size_t)H.ncoord * n_env, nu = (size_t)H.ndof * n_env;
    NSD_CK(cudaStreamSynchronize(stream));
    stage.alloc(sizeof(R) * (nq + nu));
    R* s = static_cast<R*>(stage.p);
    for (size_t i = 0; i < nq; ++i) s[i] = R(q[i]);
    for (size_t i = 0; i < nu; ++i) s[nq + i] = R(u[i]);
    NSD_CK(cudaMemcpyAsync(qs.p, s, sizeof(R) * nq, cudaMemcpyHostToDevice, stream));
    NSD_CK(cudaMemcpyAsync(us.p, s + nq, sizeof(R) * nu, cudaMemcpyHostToDevice, stream));
    NSD_CK(cudaStreamSynchronize(stream));
  }
  void get_state(double* q, double* u) override {
    const size_t nq = (size_t)H.ncoord * n_env, nu = (size_t)H.ndof * n_env;
    NSD_CK(cudaStreamSynchronize(stream));
    stage.alloc(sizeof(R) * (nq + nu));
    R* s = static_cast<R*>(stage.p);
    NSD_CK(cudaMemcpyAsync(s, qs.p, sizeof(R) * nq, cudaMemcpyDeviceToHost, stream));
    NSD_CK(cudaMemcpyAsync(s + nq, us.p, sizeof(R) * nu, cudaMemcpyDeviceToHost, stream));
    NSD_CK(cudaStreamSynchronize(stream));
    if (q)
      for (size_t i = 0; i < nq; ++i) q[i] = double(s[i]);
    if (u)
      for (size_t i = 0; i < nu; ++i) u[i] = double(s[nq + i]);
  }
  void device_state(void** q, void** u, int* dtype) override {
    *q = qs.p;
    *u = us.p;
    *dtype = sizeof(R) == 8 ? 1 : 0;
  }
  void copy_state_async(void* q, void* u) override {
    if (q) NSD_CK(cudaMemcpyAsync(q, qs.p, sizeof(R) * (size_t)H.ncoord * n_env, cudaMemcpyDefault, stream));
    if (u) NSD_CK(cudaMemcpyAsync(u, us.p, sizeof(R) * (size_t)H.ndof * n_env, cudaMemcpyDefault, stream));
  }
  long launches = 0;  // diagnostics
  void step(const void* tq, int on_device, int dtype, double h, const double* g, void* q_out = nullptr,
            void* u_out = nullptr) override {
    ++launches;
    if (!(h > 0.0)) throw NsdError(NSD_INVALID, "integrate_coordinates: h must be positive");
    BatchArgs<R> A{};
    A.T = topo.t;
    A.cfg = to_cfg(cfg);
    A.n_env = n_env;
    A.ns = ns;
    A.npairs = npairs;
    A.maxc = maxc;
    A.envs_per_block = envs_per_block;
    A.hot_in_smem = hot_in_smem ? 1 : 0;
    A.row_pool = row_pool;
    A.ptime = ptime.as<unsigned long long>();
    A.pairs = pairs.as<int2>();
    A.pair_order = porder.as<int>();
    A.shapes = shapes.as<nsd::ShapeD<R>>();
    A.jframe = topo.jframe;
    A.margin = R(margin);
    A.mu_default = R(mu_default);
    A.h = R(h);
    for (int k = 0; k < 3; ++k) A.grav[k] = R(g[k]);
    A.qs = qs.as<R>();
    A.us = us.as<R>();
    A.q_out = static_cast<R*>(q_out);
    A.u_out = static_cast<R*>(u_out);
    A.torque = nullptr;
    if (tq) {
      if (on_device) {
        A.torque = tq;
        A.torque_double = dtype;
      } else {
        const size_t n = (size_t)H.nj * n_env;
        NSD_CK(cudaStreamSynchronize(stream));  // staging buffer may still feed the previous copy
        stage.alloc(sizeof(double) * n);
        std::memcpy(stage.p, tq, sizeof(double) * n);
        NSD_CK(cudaMemcpyAsync(torque.p, stage.p, sizeof(double) * n, cudaMemcpyHostToDevice, stream));
        A.torque = torque.p;
        A.torque_double = 1;
      }
    }
    A.hot_global = hotg.as<char>();
    A.hot_bytes = plan.hot_bytes<R>();
    A.cold_r = coldr.as<R>();
    A.cold_i = coldi.as<int>();
    A.plan = plan;
    A.cand = cand.as<nsd::CandD<R>>();
    A.pair_cnt = paircnt.as<int>();
    A.nc_out = ncout.as<int>();
    A.overflow = ovf.as<int>();
    A.fin = fin.as<double>();
    A.iters = iters.as<nsd::IterOut>();
    A.jbinc_off = jbinc.as<int>();
    A.jbinc = jbinc.as<int>() + H.nb + 1;
    A.jblk = jblk.as<int4>();
    A.aborted_any = abany.as<int>();
    A.counters = ctr.as<unsigned long long>();
    A.wjinc_off = wjinc.as<int>();
    A.wjinc = warp_path ? wjinc.as<int>() + H.nb + 1 : nullptr;
    A.wplan = wplan;
    A.warp_max_obj = warp_max_obj;
    A.collide_cap = collide_cap;
    A.wsetup = wsetup.as<R>();
    A.wsetup_stride = H.ndof + 12 * H.nd3;
    A.wlam = wlam.as<R>();
    A.wptime = wptime.as<unsigned long long>();
    A.mode = 0;
    A.profile = profile ? 1 : 0;
    cudaEvent_t* ev = nullptr;
    if (time_launches && warp_path) {
      if (ev_used + 4 > evpool.size()) {
        for (int k = 0; k < 64; ++k) {
          cudaEvent_t e;
          NSD_CK(cudaEventCreate(&e));
          evpool.push_back(e);
        }
      }
      ev = &evpool[ev_used];
      ev_used += 4;
    }
    ++env_steps;
    const int epb = envs_per_block;
    const int nblk = (n_env + epb - 1) / epb;
    if (warp_path) {
      // narrow phase + setup (no shared-memory row region), the warp solver, then the
      // environments with more than 32 constraint objects through the object solver
      BatchArgs<R> A1 = A;
      A1.mode = 1;
      A1.row_pool = 0;
      A1.ptime = nullptr;
      if (ev) NSD_CK(cudaEventRecord(ev[0], stream));
      {
        Nvtx r("nsd_batch_step: narrow phase + setup (k_batch_collide)");
        NSD_CK(launch_batch_collide<R>((n_env + 3) / 4, 128, collide_smem, stream, A1));
      }
      if (ev) NSD_CK(cudaEventRecord(ev[1], stream));
      {
        Nvtx r("nsd_batch_step: newton_step, warp per env (k_batch_warp)");
        NSD_CK(launch_batch_warp<R>(mixed, (n_env + warp_epb - 1) / warp_epb, 32 * warp_epb, warp_smem, stream, A));
      }
      if (ev) NSD_CK(cudaEventRecord(ev[2], stream));
      A.mode = 2;
      {
        Nvtx r("nsd_batch_step: newton_step, large envs (k_batch_sub mode 2)");
        NSD_CK(launch_batch_sub<R>(16, nblk, 16 * epb, smem_bytes, stream, A));
      }
      if (ev) NSD_CK(cudaEventRecord(ev[3], stream));
      return;
    }
    if (team_threads <= 32) {
      const int thr = team_threads * epb;
      NSD_CK(launch_batch_sub<R>(team_threads, nblk, thr, smem_bytes, stream, A));
    } else {
      NSD_CK(launch_batch_block<R>(n_env, team_threads, smem_bytes, stream, A));
    }
  }
  void results(int* nc, int* ab, double* fres, nsd_iter_stats* its) override {
    std::vector<int> hn(n_env), ho(n_env);
    std::vector<double> hf(8 * (size_t)n_env);
    std::vector<int> ha(n_env);
    NSD_CK(cudaMemcpyAsync(hn.data(), ncout.p, sizeof(int) * n_env, cudaMemcpyDeviceToHost, stream));
    NSD_CK(cudaMemcpyAsync(ho.data(), ovf.p, sizeof(int) * n_env, cudaMemcpyDeviceToHost, stream));
    NSD_CK(cudaMemcpyAsync(ha.data(), abany.p, sizeof(int) * n_env, cudaMemcpyDeviceToHost, stream));
    // overflow and abort are sticky over the steps since the previous call: read, then clear
    NSD_CK(cudaMemsetAsync(ovf.p, 0, sizeof(int) * n_env, stream));
    NSD_CK(cudaMemsetAsync(abany.p, 0, sizeof(int) * n_env, stream));
    NSD_CK(cudaMemcpyAsync(hf.data(), fin.p, sizeof(double) * 8 * n_env, cudaMemcpyDeviceToHost, stream));
    std::vector<nsd::IterOut> hi;
    const int N = cfg.newton_iterations;
    if (its) {
      hi.resize((size_t)N * n_env);
      NSD_CK(cudaMemcpyAsync(hi.data(), iters.p, sizeof(nsd::IterOut) * hi.size(), cudaMemcpyDeviceToHost, stream));
    }
    NSD_CK(cudaStreamSynchronize(stream));
    int overflow_env = -1;
    for (int e = 0; e < n_env; ++e) {
      if (nc) nc[e] = hn[e];
      if (ab) ab[e] = ha[e] != 0;
      if (fres) fres[e] = hf[8 * e];
      if (ho[e] && overflow_env < 0) overflow_env = e;
    }
    if (its)
      for (size_t i = 0; i < hi.size(); ++i) {
        its[i].residual_inf = hi[i].residual_inf;
        its[i].merit_l2 = hi[i].merit_l2;
        its[i].comp_error_max = hi[i].comp_error_max;
        its[i].cone_violation_max = hi[i].cone_violation_max;
        its[i].step_size = hi[i].step_size;
        its[i].linear_residual = hi[i].linear_residual;
        its[i].linear_iterations = hi[i].linear_iterations;
        its[i].linear_breakdown = hi[i].linear_breakdown;
      }
    if (overflow_env >= 0)
      throw NsdError(NSD_INVALID, "env " + std::to_string(overflow_env) + " produced " +
                                      std::to_string(ho[overflow_env]) + " contacts > max_contacts " +
                                      std::to_string(maxc));
  }
  // [0] PCR iterations summed over envs and steps, [1] cycles inside the PCR loops
  // (warp path, profile on), [2] cycles per env step (same), [3] env-steps; read and reset
  void counters(unsigned long long* out) override {
    NSD_CK(cudaStreamSynchronize(stream));
    unsigned long long c4[4];
    NSD_CK(cudaMemcpy(c4, ctr.p, sizeof(c4), cudaMemcpyDeviceToHost));
    for (int k = 0; k < 3; ++k) out[k] = c4[k];
    out[3] = static_cast<unsigned long long>(env_steps) * n_env;
    out[8] = c4[3];
    env_steps = 0;
    NSD_CK(cudaMemset(ctr.p, 0, sizeof(unsigned long long) * 4));
    double us[3] = {0.0, 0.0, 0.0};
    for (size_t i = 0; i + 4 <= ev_used; i += 4)
      for (int k = 0; k < 3; ++k) {
        float ms = 0.f;
        NSD_CK(cudaEventElapsedTime(&ms, evpool[i + k], evpool[i + k + 1]));
        us[k] += 1000.0 * ms;
      }
    for (int k = 0; k < 3; ++k) out[4 + k] = static_cast<unsigned long long>(us[k] * 1000.0 + 0.5);  // ns
    out[7] = ev_used / 4;
    ev_used = 0;
  }
  void set_profile(int on) override {
    profile = (on & 1) != 0;
    time_launches = (on & 2) != 0;
  }
  void contacts(int env, nsd_contact* out, int* n) override {
    if (env < 0 || env >= n_env) throw NsdError(NSD_INVALID, "env out of range");
    int nc = 0;
    NSD_CK(cudaMemcpyAsync(&nc, ncout.as<int>() + env, sizeof(int), cudaMemcpyDeviceToHost, stream));
    NSD_CK(cudaStreamSynchronize(stream));
    *n = nc;
    if (!out || nc == 0) return;
    std::vector<int> cb(2 * nc), cf(nc);
    std::vector<R> cg(17 * (size_t)nc), lam(H.rows_static + 3 * (size_t)nc);
    const R* cr = coldr.as<R>() + (size_t)env * plan.coldR;
    const int* ci = coldi.as<int>() + (size_t)env * plan.coldI;
    NSD_CK(cudaMemcpyAsync(cb.data(), ci + plan.xcbody, sizeof(int) * 2 * nc, cudaMemcpyDeviceToHost, stream));
    NSD_CK(cudaMemcpyAsync(cf.data(), ci + plan.cfeat, sizeof(int) * nc, cudaMemcpyDeviceToHost, stream));
    NSD_CK(cudaMemcpyAsync(cg.data(), cr + plan.cgeo, sizeof(R) * 17 * nc, cudaMemcpyDeviceToHost, stream));
    NSD_CK(cudaMemcpyAsync(lam.data(), cr + plan.xlam, sizeof(R) * lam.size(), cudaMemcpyDeviceToHost, stream));
    NSD_CK(cudaStreamSynchronize(stream));
    for (int c = 0; c < nc; ++c) {
      nsd_contact& k = out[c];
      std::memset(&k, 0, sizeof(k));
      k.body_a = cb[2 * c];
      k.body_b = cb[2 * c + 1];
      k.feature = cf[c];
      for (int i = 0; i < 3; ++i) {
        k.local_a[i] = cg[17 * c + i];
        k.local_b[i] = cg[17 * c + 3 + i];
        k.normal[i] = cg[17 * c + 6 + i];
        k.d1[i] = cg[17 * c + 9 + i];
        k.d2[i] = cg[17 * c + 12 + i];
      }
      k.thickness = cg[17 * c + 15];
      k.mu = cg[17 * c + 16];
      k.lambda_n = lam[H.rows_static + c];
      k.lambda_f[0] = lam[H.rows_static + nc + 2 * c];
      k.lambda_f[1] = lam[H.rows_static + nc + 2 * c + 1];
    }
  }
};

// ================================================================== C ABI
struct nsd_solver {
  std::unique_ptr<SolverBase> impl;
};
struct nsd_batch {
  std::unique_ptr<BatchBase> impl;
};

extern "C" {

const char* nsd_last_error(void) { return g_err.c_str(); }

void nsd_config_default(nsd_config* c, int32_t precision) {
  c->newton_iterations = 8;
  c->step_fraction = 0.75;
  c->epsilon_reg = 1e-6;
  c->geometric_stiffness = 1;
  c->r_strategy = 2;
  c->ncp_kind = 1;
  c->linear_method = 3;
  c->linear_max_iterations = 40;
  c->linear_tolerance = 1e-10;
  c->preconditioner = 1;
  c->newton_tolerance = 1e-6;
  c->line_search = 0;
  c->precision = precision;
}

int32_t nsd_count_rows(const nsd_topology* topo, int32_t n_contacts) {
  if (!topo) return -1;
  int n = 0;
  for (int j = 0; j < topo->n_joints; ++j) n += nsd::joint_nrows(topo->joint_kind[j]);
  for (int e = 0; e < topo->n_tets; ++e)  // 3 per Neo-Hookean tet, 6 per linear tet (newton.cpp:32-33)
    n += (static_cast<int>(topo->tet_material[4 * e + 3]) & 2) ? 6 : 3;
  return n + 3 * n_contacts;
}

int nsd_create(const nsd_topology* topo, const nsd_config* cfg, int32_t device, nsd_solver** out) {
  return guarded([&] {
    if (!topo || !cfg || !out) throw NsdError(NSD_INVALID, "null argument");
    check_cfg(*cfg);
    auto* s = new nsd_solver();
    try {
      // one fp64 engine for both precisions: fp32 stores the operator's J/C
      // coefficients in fp32 (NSD_OP32 kernels, nsd_k_single32.cu), state and arithmetic stay fp64
      s->impl.reset(new Solver<double>(*topo, *cfg, device));
    } catch (...) {
      delete s;
      throw;
    }
    *out = s;
    return NSD_OK;
  });
}

int nsd_set_config(nsd_solver* s, const nsd_config* cfg) {
  return guarded([&] {
    if (!s || !cfg) throw NsdError(NSD_INVALID, "null argument");
    check_cfg(*cfg);
    s->impl->set_cfg(*cfg);
    return NSD_OK;
  });
}

int nsd_step(nsd_solver* s, const nsd_step_in* in, nsd_step_out* out) {
  return guarded([&] {
    if (!s) throw NsdError(NSD_INVALID, "null solver");
    return s->impl->step(in, out);
  });
}

double nsd_last_step_ms(const nsd_solver* s) { return s ? s->impl->last_ms : 0.0; }

int nsd_destroy(nsd_solver* s) {
  delete s;
  return NSD_OK;
}

int nsd_batch_create(const nsd_topology* topo, int32_t n_shapes, const nsd_shape* shapes, double margin,
                     double mu_default, const nsd_config* cfg, int32_t n_env, int32_t max_contacts, int32_t device,
                     nsd_batch** out) {
  return guarded([&] {
    if (!topo || !cfg || !out || (n_shapes > 0 && !shapes)) throw NsdError(NSD_INVALID, "null argument");
    check_cfg(*cfg);
    auto* b = new nsd_batch();
    try {
      // fp32 is the mixed-precision mode: fp64 state, assembly, Newton update and
      // reductions; the PCR operator's data and row vectors in fp32 (warp path)
      b->impl.reset(new Batch<double>(*topo, n_shapes, shapes, margin, mu_default, *cfg, n_env, max_contacts, device,
                                      cfg->precision == NSD_FP32));
    } catch (...) {
      delete b;
      throw;
    }
    *out = b;
    return NSD_OK;
  });
}

int nsd_batch_set_state(nsd_batch* b, const double* q, const double* u) {
  return guarded([&] {
    if (!b || !q || !u) throw NsdError(NSD_INVALID, "null argument");
    b->impl->set_state(q, u);
    return NSD_OK;
  });
}

int nsd_batch_get_state(nsd_batch* b, double* q, double* u) {
  return guarded([&] {
    if (!b) throw NsdError(NSD_INVALID, "null argument");
    b->impl->get_state(q, u);
    return NSD_OK;
  });
}

int nsd_batch_set_stream(nsd_batch* b, void* stream) {
  return guarded([&] {
    if (!b) throw NsdError(NSD_INVALID, "null argument");
    if (b->impl->own_stream && b->impl->stream) cudaStreamDestroy(b->impl->stream);
    if (stream) {
      b->impl->stream = static_cast<cudaStream_t>(stream);
      b->impl->own_stream = false;
    } else {
      NSD_CK(cudaStreamCreateWithFlags(&b->impl->stream, cudaStreamNonBlocking));
      b->impl->own_stream = true;
    }
    return NSD_OK;
  });
}

int nsd_batch_step(nsd_batch* b, const double* joint_torque, int32_t torque_on_device, double h,
                   const double gravity[3]) {
  return guarded([&] {
    if (!b || !gravity) throw NsdError(NSD_INVALID, "null argument");
    b->impl->step(joint_torque, torque_on_device, 1, h, gravity);
    return NSD_OK;
  });
}

int nsd_batch_step_device(nsd_batch* b, const void* joint_torque_dev, int32_t dtype, double h,
                          const double gravity[3]) {
  return guarded([&] {
    if (!b || !gravity) throw NsdError(NSD_INVALID, "null argument");
    b->impl->step(joint_torque_dev, 1, dtype, h, gravity);
    return NSD_OK;
  });
}

// A pointer the device can dereference: device or managed memory as is, pinned host
// memory through its device mapping (UVA: the same address for cudaHostAlloc'd memory).
static void* device_view(const void* p, const char* what) {
  if (!p) return nullptr;
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    throw NsdError(NSD_INVALID, std::string(what) + ": not device memory or pinned host memory");
  }
  if (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged) return const_cast<void*>(p);
  if (at.type == cudaMemoryTypeHost && at.devicePointer) return at.devicePointer;
  throw NsdError(NSD_INVALID, std::string(what) + ": pageable host memory (pin it, e.g. cudaHostAlloc)");
}

int nsd_batch_step_mapped(nsd_batch* b, const void* joint_torque, int32_t dtype, void* q_out, void* u_out, double h,
                          const double gravity[3]) {
  return guarded([&] {
    if (!b || !gravity) throw NsdError(NSD_INVALID, "null argument");
    if (dtype != 0 && dtype != 1) throw NsdError(NSD_INVALID, "dtype must be 0 (float) or 1 (double)");
    const void* tq = device_view(joint_torque, "joint_torque");
    void* qo = device_view(q_out, "q_out");
    void* uo = device_view(u_out, "u_out");
    b->impl->step(tq, 1, dtype, h, gravity, qo, uo);
    return NSD_OK;
  });
}

int nsd_batch_sync(nsd_batch* b) {
  return guarded([&] {
    if (!b) throw NsdError(NSD_INVALID, "null argument");
    NSD_CK(cudaStreamSynchronize(b->impl->stream));
    return NSD_OK;
  });
}

int nsd_batch_results(nsd_batch* b, int32_t* n_contacts, int32_t* aborted, double* final_residual_inf,
                      nsd_iter_stats* iters) {
  return guarded([&] {
    if (!b) throw NsdError(NSD_INVALID, "null argument");
    b->impl->results(n_contacts, aborted, final_residual_inf, iters);
    return NSD_OK;
  });
}

int nsd_batch_contacts(nsd_batch* b, int32_t env, nsd_contact* out, int32_t* n) {
  return guarded([&] {
    if (!b || !n) throw NsdError(NSD_INVALID, "null argument");
    b->impl->contacts(env, out, n);
    return NSD_OK;
  });
}

int nsd_batch_device_state(nsd_batch* b, void** q_dev, void** u_dev, int32_t* dtype) {
  return guarded([&] {
    if (!b || !q_dev || !u_dev || !dtype) throw NsdError(NSD_INVALID, "null argument");
    b->impl->device_state(q_dev, u_dev, dtype);
    return NSD_OK;
  });
}

int nsd_batch_copy_state_async(nsd_batch* b, void* q_dst, void* u_dst) {
  return guarded([&] {
    if (!b) throw NsdError(NSD_INVALID, "null argument");
    b->impl->copy_state_async(q_dst, u_dst);
    return NSD_OK;
  });
}

int nsd_batch_counters(nsd_batch* b, uint64_t* out) {
  return guarded([&] {
    if (!b || !out) throw NsdError(NSD_INVALID, "null argument");
    unsigned long long v[9];
    b->impl->counters(v);
    for (int i = 0; i < 9; ++i) out[i] = v[i];
    return NSD_OK;
  });
}

int nsd_batch_profile(nsd_batch* b, int32_t enable) {
  return guarded([&] {
    if (!b) throw NsdError(NSD_INVALID, "null argument");
    b->impl->set_profile(enable);
    return NSD_OK;
  });
}

int nsd_batch_info(const nsd_batch* b, int32_t* info) {
  if (!b || !info) return NSD_INVALID;
  for (int i = 0; i < 6; ++i) info[i] = b->impl->info[i];
  return NSD_OK;
}

int nsd_batch_destroy(nsd_batch* b) {
  delete b;
  return NSD_OK;
}

}  // extern "C"
