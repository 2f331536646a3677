/* nsdyn_gpu.h — C ABI of the B200-native non-smooth Newton step.
 *
 * Drop-in boundary for the reference's hot path
 *   SolveReport nsdyn::newton_step(const StepContext&, const NewtonConfig&)
 *   (/root/reference/proj/include/nsdyn/newton.h:116-118, src/newton.cpp:321-418)
 * plus the batched many-environment path and the world-level
 * builders used by bench.py. Plain C types only: int32 ids, double state,
 * host pointers. Every call returns an int status (NSD_OK ... NSD_UNSUPPORTED);
 * nsd_last_error() gives the text of the last failure on the calling thread.
 *
 * Semantics mirrored from the reference:
 *   - units: multipliers are h-scaled impulses (constraints.h:46), telemetry
 *     reports forces lambda/h (newton.cpp:83-85);
 *   - NaN in the Newton update rolls q,u back to the step start and reports
 *     aborted (newton.cpp:362-369) -> status NSD_ABORTED, outputs still filled;
 *   - invalid input (h <= 0, bad body index, dimension mismatch) -> NSD_INVALID
 *     where the reference throws std::invalid_argument (bodies.cpp:80,
 *     constraints.cpp:142-144, solvers.cpp:188-190);
 *   - PCR breakdown is flagged in the iteration stats, never an error.
 * Handles are not thread-safe; distinct handles may be used concurrently
 * ("scenes step concurrently without shared mutable state").
 */
#ifndef NSDYN_GPU_H
#define NSDYN_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NSD_OK 0
#define NSD_INVALID 1
#define NSD_ABORTED 2
#define NSD_CUDA_ERROR 3
#define NSD_UNSUPPORTED 4

#define NSD_FP32 0
#define NSD_FP64 1

/* NewtonConfig + LinearSolverConfig (newton.h:12-23, solvers.h:11-16). */
typedef struct nsd_config {
  int32_t newton_iterations;     /* default 8 */
  double step_fraction;          /* damped Newton t, default 0.75 */
  double epsilon_reg;            /* default 1e-6 */
  int32_t geometric_stiffness;   /* default 1 */
  int32_t r_strategy;            /* 0 Identity, 1 TimestepSquared, 2 EffectiveMass (default) */
  int32_t ncp_kind;              /* 0 MinimumMap, 1 FischerBurmeister (default) */
  int32_t linear_method;         /* 0 Jacobi, 1 Gauss-Seidel, 2 PCG, 3 PCR (default); batches: PCR only */
  int32_t linear_max_iterations; /* default 40 */
  double linear_tolerance;       /* absolute residual 2-norm, default 1e-10 */
  int32_t preconditioner;        /* 0 None, 1 Diagonal (default) */
  double newton_tolerance;       /* convergence classification only, default 1e-6 */
  int32_t line_search;           /* merit backtracking, frictionless scenes only */
  int32_t precision;             /* NSD_FP64, or NSD_FP32: mixed mode (fp64 state and arithmetic, fp32 operator coefficients) */
} nsd_config;

/* Fills the reference defaults (newton.h:12-23) with the given precision. */
void nsd_config_default(nsd_config* cfg, int32_t precision);

/* Static scene data, uploaded once (GeneralizedState bodies, JointSpec,
 * MeshBinding/TetMeshElements: bodies.h:11-43, constraints.h:72-86,
 * materials.h:10-77, newton.h:26-29). */
typedef struct nsd_topology {
  int32_t n_bodies;
  const int32_t* body_type;    /* 0 particle (3 dof / 3 coord), 1 rigid (6 dof / 7 coord) */
  const double* body_mass;
  const double* body_inertia;  /* 9 per body, row-major, body frame (rigid only) */
  int32_t n_joints;
  const int32_t* joint_kind;   /* 0 FixedPoint, 1 Revolute, 2 Prismatic, 3 BendSpring */
  const int32_t* joint_body;   /* 2 per joint: body_a, body_b (-1 = world) */
  const double* joint_frame;   /* 21 per joint: anchor_a, anchor_b, axis_a, axis_a2, axis_b1, axis_b2, rest_dots */
  const double* joint_param;   /* 2 per joint: compliance, stiffness */
  int32_t n_tets;              /* all meshes, mesh-major = row-layout order */
  const int32_t* tet_body;     /* 4 per tet: global body index of each vertex particle */
  const double* tet_dm_inv;    /* 9 per tet, row-major */
  const double* tet_volume;
  const double* tet_material;  /* 4 per tet: c1 = mu/2, d1 = lambda/2, alpha, flags (1 diagonal compliance,
                                  2 linear co-rotational: 6 rows per tet, 6x6 compliance; one model per scene) */
} nsd_topology;

/* ContactConstraint (constraints.h:40-50); body -1 = world point in local. */
typedef struct nsd_contact {
  int32_t body_a, body_b, feature, pad;
  double local_a[3], local_b[3], normal[3], d1[3], d2[3];
  double thickness, mu;
  double lambda_n, lambda_f[2]; /* written back by nsd_step (newton.cpp:74-78) */
  double pad2[2];
} nsd_contact;

/* NewtonIterationStats (newton.h:45-54). */
typedef struct nsd_iter_stats {
  double residual_inf, merit_l2, comp_error_max, cone_violation_max, step_size;
  double linear_residual;
  int32_t linear_iterations, linear_breakdown;
} nsd_iter_stats;

typedef struct nsd_step_in {
  const double* q;           /* num_coord, packed (3 per particle, 7 per rigid: pos, quat wxyz) */
  const double* u;           /* num_dof, packed */
  int32_t n_contacts;
  const nsd_contact* contacts;
  double h;
  double gravity[3];
  const double* f_extra;     /* optional num_dof generalized force (extension hook) */
  const double* joint_frame; /* optional 21*n_joints update (driven anchors) */
} nsd_step_in;

typedef struct nsd_step_out {
  double* q;                 /* num_coord (may alias in.q) */
  double* u;                 /* num_dof  (may alias in.u) */
  double* lambda;            /* optional: n_rows multipliers (row layout of make_layout) */
  nsd_contact* contacts;     /* optional: lambda_n / lambda_f written (may alias in.contacts) */
  nsd_iter_stats* iters;     /* optional: newton_iterations entries */
  double* linear_history;    /* optional: newton_iterations * (linear_max_iterations + 1) */
  int32_t* linear_history_len; /* optional: newton_iterations */
  double* contact_telemetry; /* optional: 6 per contact: gap, lambda_n, |lambda_f|, mu, |v_t|, lambda_f.v_t */
  /* scalar results */
  int32_t n_iterations, n_rows;
  double final_residual_inf, final_comp_error, final_cone_violation, min_gap, min_diag_shift;
  int32_t aborted, converged;
  /* optional: newton_iterations x (n_contacts + n_tets + num_dof + 1) decision bytes
   * per Newton iteration: per contact bit0 normal J row kept, bit1
   * friction active, bit2 W capped at 1e12, bit3 min-map stick branch (W = 0), bit4 NCP branch (FB origin /
   * min-map c <= r lambda); per tet bit0 PSD projection, bit1 diagonal compliance
   * fallback; per dof bit0 GS secant skipped, bit1 GS clamp, bit2 rigid dof zeroed
   * (GS active iterations); last byte the PCR exit: 0 budget, 1 tolerance, 2 monotone
   * guard, 3 breakdown, 4 no rows. */
  uint8_t* decisions;
} nsd_step_out;

typedef struct nsd_solver nsd_solver;

const char* nsd_last_error(void);

/* count_rows (newton.h:114): joints 3/5/5/2, 3 per Neo-Hookean / 6 per linear tet, 3 per contact. */
int32_t nsd_count_rows(const nsd_topology* topo, int32_t n_contacts);

int nsd_create(const nsd_topology* topo, const nsd_config* cfg, int32_t device, nsd_solver** out);
int nsd_set_config(nsd_solver* s, const nsd_config* cfg);
/* newton_step: synchronous, one scene (newton.cpp:321-418). */
int nsd_step(nsd_solver* s, const nsd_step_in* in, nsd_step_out* out);
/* Device time in ms of the last nsd_step's kernel(s) (CUDA events). */
double nsd_last_step_ms(const nsd_solver* s);
int nsd_destroy(nsd_solver* s);

/* ---------------- batched many-environment path (one topology, many states) */
typedef struct nsd_shape {  /* AttachedShape (collision.h:8-27) */
  int32_t body, kind;       /* kind: 0 HalfSpace, 1 Sphere, 2 Box */
  double normal[3], offset, radius, half_extents[3], thickness, mu;
} nsd_shape;

typedef struct nsd_batch nsd_batch;

/* n_env environments share `topo` and `shapes`; contacts are detected on the
 * device each step (collision.cpp:239-297 semantics) with at most
 * max_contacts per env (exceeding it is reported, never truncated silently). */
int nsd_batch_create(const nsd_topology* topo, int32_t n_shapes, const nsd_shape* shapes, double margin,
                     double mu_default, const nsd_config* cfg, int32_t n_env, int32_t max_contacts,
                     int32_t device, nsd_batch** out);
/* q: n_env*num_coord, u: n_env*num_dof (host doubles). */
int nsd_batch_set_state(nsd_batch* b, const double* q, const double* u);
int nsd_batch_get_state(nsd_batch* b, double* q, double* u);
/* Uses the caller's CUDA stream (cudaStream_t) for all batch work; NULL = own stream. */
int nsd_batch_set_stream(nsd_batch* b, void* stream);
/* One step_world for every env (scene.cpp:709-732): detect + newton_step.
 * joint_torque: optional n_env*n_joints torques applied about revolute axes
 * (extension hook); host pointer if torque_on_device == 0, else device pointer.
 * Asynchronous on the batch stream. */
int nsd_batch_step(nsd_batch* b, const double* joint_torque, int32_t torque_on_device, double h,
                   const double gravity[3]);
/* Device-resident variant: torques already on device as float or double array
 * of n_env*n_joints (dtype 0 float, 1 double), NULL for passive. */
int nsd_batch_step_device(nsd_batch* b, const void* joint_torque_dev, int32_t dtype, double h,
                          const double gravity[3]);
int nsd_batch_sync(nsd_batch* b);
/* Per-env results: n_contacts[n_env] and final_residual_inf[n_env] of the last
 * step; aborted[n_env] = 1 if the env rolled back (newton.cpp:362-369) in ANY
 * step since the previous call; iters: n_env*newton_iterations of the last step
 * (optional). A contact overflow (more than max_contacts) in any step since the
 * previous call is NSD_INVALID. Overflow and abort flags are cleared by the call. */
int nsd_batch_results(nsd_batch* b, int32_t* n_contacts, int32_t* aborted, double* final_residual_inf,
                      nsd_iter_stats* iters);
/* Contact list of one env from the last step (count in *n). */
int nsd_batch_contacts(nsd_batch* b, int32_t env, nsd_contact* out, int32_t* n);
/* Device pointers of the packed state (for zero-copy consumers). */
int nsd_batch_device_state(nsd_batch* b, void** q_dev, void** u_dev, int32_t* dtype);
/* Enqueues (no sync) a copy of the packed state in the batch precision
 * (float or double, see nsd_batch_device_state) to q_dst / u_dst (pinned host
 * or device memory); either may be NULL. */
int nsd_batch_copy_state_async(nsd_batch* b, void* q_dst, void* u_dst);
/* nsd_batch_step_device with the transfers inside the step: joint_torque
 * (n_env*n_joints, dtype 0 float / 1 double, NULL = passive) and q_out / u_out
 * (n_env*num_coord / n_env*num_dof in the batch precision, either may be NULL)
 * may be pinned host memory (cudaHostAlloc, or torch pin_memory): the step
 * kernel reads each env's torques and writes its final state over the bus,
 * overlapped with the other envs' compute. Device pointers are accepted too;
 * pageable host memory is NSD_INVALID. q_out / u_out are complete once the
 * batch stream has passed the step (nsd_batch_sync). The device state is
 * updated as by nsd_batch_step_device. Replaces, in the reference's RL loop,
 * the per-step torque upload + state read-back around step_world
 * (scene.cpp:709-732 per env). */
int nsd_batch_step_mapped(nsd_batch* b, const void* joint_torque, int32_t dtype, void* q_out, void* u_out, double h,
                          const double gravity[3]);
int nsd_batch_info(const nsd_batch* b, int32_t* info /* [n_env, num_coord, num_dof, n_joints, max_rows, team_threads] */);
/* Counters since the previous call (read and reset; synchronises the stream),
 * out[9]: [0] PCR iterations run, summed over envs, Newton iterations and steps
 * (the roofline numerator counts these); [1] clock64 cycles spent inside the
 * PCR loops and [2] cycles per env step, both summed over envs (profile bit 0,
 * warp path); [3] env-steps; [4..6] nanoseconds between CUDA events recorded on
 * the batch stream around the step's narrow-phase launch, warp-solver launch and
 * large-env launch, summed over [7] timed steps (profile bit 1, warp path);
 * [8] PCR iterations x the env's contact count, summed like [0] (the per-env
 * algorithmic bytes of one PCR iteration are affine in the contact count). */
int nsd_batch_counters(nsd_batch* b, uint64_t* out);
/* profile flags: bit 0 in-kernel cycle counters, bit 1 per-launch CUDA events. */
int nsd_batch_profile(nsd_batch* b, int32_t flags);
int nsd_batch_destroy(nsd_batch* b);

/* ---------------- builders (scene.cpp:802-935 style) */
typedef struct nsd_scene nsd_scene;
/* name: "c1".."c5", "box_on_plane", "heavy_stack", "incline:<deg>:<mu>", ... */
int nsd_scene_build(const char* name, uint32_t seed, nsd_scene** out);
/* The reference's JSON scene format. nsd_scene_parse: parse_scene + build_world
 * (scene.cpp:293-470, 587-707): fully validated, unknown keys rejected; on error
 * NSD_INVALID and the reference's message ("scene error at bodies[0].mass: must
 * be positive", "scene syntax error: ...") in err (NUL-terminated, truncated to
 * err_capacity). nsd_scene_serialize: serialize_scene (scene.cpp:472-556), the
 * document with sorted keys and 2-space indentation; *length = its size without
 * the NUL, written to buf when capacity > length (buf NULL: size query). Scenes
 * from nsd_scene_build serialize too (product-only mesh extensions omitted). */
int nsd_scene_parse(const char* json, nsd_scene** out, char* err, int32_t err_capacity);
int nsd_scene_serialize(const nsd_scene* s, char* buf, int64_t capacity, int64_t* length);
/* dims: n_bodies, num_dof, num_coord, n_joints, n_tets, n_shapes, newton_iterations, linear_max_iterations */
int nsd_scene_dims(const nsd_scene* s, int32_t* dims);
int nsd_scene_topology(const nsd_scene* s, nsd_topology* topo); /* pointers valid while s lives */
int nsd_scene_shapes(const nsd_scene* s, nsd_shape* shapes, double* margin, double* mu_default);
int nsd_scene_state(const nsd_scene* s, double* q, double* u);
int nsd_scene_config(const nsd_scene* s, nsd_config* cfg, double* h, double* gravity);
int nsd_scene_destroy(nsd_scene* s);
/* Current joint frames (21 per joint, nsd_topology layout; driven anchors move). */
int nsd_scene_joint_frames(const nsd_scene* s, double* frames);
/* Moves the world-side anchors of driven joints by h * anchor_velocity
 * (step_world's first statement, scene.cpp:710-716). */
int nsd_scene_advance_anchors(nsd_scene* s);
/* Caller side of step_world on the host (scene.cpp:717-721): u~ from (q, u,
 * optional f_extra), narrow phase over the scene's shapes plus the particle
 * generators, predicted-gap rule, canonical order (collision.cpp:239-297).
 * *n receives the contact count; NSD_INVALID if it exceeds capacity. */
int nsd_scene_detect(const nsd_scene* s, const double* q, const double* u, const double* f_extra, int32_t capacity,
                     nsd_contact* out, int32_t* n);
/* Initial states of n copies of a seeded builder (seed0 .. seed0+n-1), e.g. the
 * per-environment C5 ants: q n*num_coord, u n*num_dof. */
int nsd_scene_batch_state(const char* name, uint32_t seed0, int32_t n, double* q, double* u);

#ifdef __cplusplus
}
#endif

#endif /* NSDYN_GPU_H */
