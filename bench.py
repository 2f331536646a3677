#!/usr/bin/env python3
"""Benchmark: batched non-smooth Newton step, C5 workload (ant environments).

One "step" = one step_world for every environment on the GPU: device narrow
phase (sphere/box vs half-space and body pairs) + the full non-smooth Newton
solve (4 Newton x 10 PCR, Fischer-Burmeister, effective-mass r, friction) +
integration. Three launches per step: the narrow-phase/setup launch
(k_batch_sub, mode 1), the warp-per-env solver (k_batch_warp, the dominant
kernel) and the launch that solves envs with more than 32 constraint objects
(k_batch_sub, mode 2; exits at once when there are none).

  value   env-steps/s, actions pre-staged in HBM, L2 flushed between steps,
          device time (CUDA events) summed over exactly K steps, max over ranks
  e2e     same metric through the C ABI with host actions: per step the joint
          torques from pinned memory in, (q, u) to pinned memory out. Headline:
          nsd_batch_step_mapped (the step kernel moves those bytes over the bus
          itself, overlapped with compute); copy_path_value: H2D copy + step +
          D2H copy. Both replay the same steps and must end in the same state.
  dtype   f64 by default: the precision the reference computes in and the one
          whose oracle parity is proven (1e-8 over 25 steps, tests/test_gpu_batch.py);
          the other precision (f32 performance mode) is measured too and
          reported under "other_precision" (--no-alt skips it)
  --impl reference   the reference's CPU path: the oracle restatement of
          nsdyn::step_world (oracle/, the reference itself does not build here),
          OpenMP over environments on all host cores.

  roofline  SURVEY §8(d) algorithmic bytes of the PCR iterations actually run
          (nsd_batch_counters: sum of linear_iterations, and of iterations x the
          env's contact count — B_CR is affine in it) over the dominant kernel's
          CUDA-event time inside the timed region ("frac"); also over the whole
          step ("frac_step") and over the PCR loops alone ("frac_cr_loop": the
          kernel time x the in-kernel clock64 share of the PCR loops, measured in
          a separate untimed replay of the same steps).

Multi-GPU: one process per GPU, each rank owns envs [rank*E, (rank+1)*E) with
global-env-id seeds; no collective on the data path; "scaling":
"weak". `bench.py --gpus N` without a torchrun environment re-launches itself
under torch.distributed.run with N processes (both arms).
"""
import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
HBM_FALLBACK = 6650.0


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--envs", type=int, default=4096, help="environments per GPU")
    p.add_argument("--precision", default="fp64", choices=["fp32", "fp64"])
    p.add_argument("--passive", action="store_true", help="no joint torques (pure reference semantics)")
    p.add_argument("--team", type=int, default=0, help="threads per env team (32 = warp, 64/128 = CTA)")
    p.add_argument("--max-contacts", type=int, default=48)
    p.add_argument("--cpu-seconds", type=float, default=12.0, help="target CPU baseline sample length")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-alt", action="store_true", help="skip the secondary-precision measurement")
    p.add_argument("--no-parity-sample", action="store_true", help="skip the end-of-run oracle check of 64 envs")
    p.add_argument("--no-scenes", action="store_true", help="skip the C1-C4 single-scene summary")
    p.add_argument("--workload", default="c5",
                   help="c5 (default: batched ants, the headline) or one single scene (c1, c2, c3, c4, c2:6, ...) "
                        "stepped through World.step (host detect + GPU newton_step)")
    return p.parse_args()


def maybe_relaunch(args):
    """--gpus N > 1 outside torchrun: re-exec under torch.distributed.run (N ranks)."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    os.execv(sys.executable, cmd)


def dist_info():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region: the
    sampler is started and waited for (its first line) before the region opens,
    and only samples taken between begin() and end() are reported."""

    def __init__(self, device):
        self.device, self.samples, self.proc, self.thread = device, [], None, None
        self.t0 = self.t1 = None

    def start(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()
        deadline = time.time() + 5.0
        while not self.samples and time.time() < deadline:  # nvidia-smi is up and sampling
            time.sleep(0.01)

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 6:
                self.samples.append((time.time(), parts))

    def begin(self):
        self.t0 = time.time()

    def end(self):
        self.t1 = time.time()

    def stop(self):
        if self.t1 is None:
            self.end()
        time.sleep(0.05)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        t0 = self.t0 if self.t0 is not None else 0.0
        inside = [p for t, p in self.samples if t0 <= t <= self.t1 + 0.02]
        sm = [float(s[0]) for s in inside if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in inside if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in inside for i in range(4) if "Active" in s[2 + i] and "Not" not in s[2 + i]})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(inside)}


def hbm_peak():
    try:
        with open(PEAKS) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return HBM_FALLBACK, "fallback"


def b_cr_bytes(n_contacts, nj_rows=40, n_joint_nnz=384, n_joints=8, dof=54, rigid=9, value_bytes=4):
    """SURVEY §8(d) algorithmic bytes of one CR iteration for one ant env:
    B_CR = 2(vZ + 4X) + v n_C + 2vD + v D_particle + 7v B_rigid + 13 v R
    (fp32: v = 4 -> 2(4Z+4X) + 4n_C + 8D + 4D_p + 28B_rigid + 52R); affine in nc."""
    nc = np.asarray(n_contacts, dtype=np.float64)
    R = nj_rows + 3 * nc
    Z = n_joint_nnz + 18 * nc
    X = 2 * n_joints + 2 * nc
    n_C = R
    v = value_bytes
    return 2 * (v * Z + 4 * X) + v * n_C + 2 * v * dof + 7 * v * rigid + 13 * v * R


def scene_b_cr(dims, topo, n_contacts, contact_bodies, value_bytes=8):
    """SURVEY §8(d) B_CR of one PCR iteration of a single scene, from its exact
    structure: Z (J nonzeros), X (int32 ids), n_C (C entries), R, D, D_particle,
    B_rigid. contact_bodies: (body_a, body_b) per contact (-1 = world)."""
    bt = np.asarray(topo.a["body_type"])
    side = lambda b: 0 if b < 0 else (6 if bt[b] == 1 else 3)
    Z = X = n_C = R = 0
    kinds, jb = np.asarray(topo.a["joint_kind"]), np.asarray(topo.a["joint_body"]).reshape(-1, 2)
    for k, (a, b) in zip(kinds, jb):
        npnt = 3 if k <= 1 else (2 if k == 2 else 0)
        nr = 2 if k == 3 else (3 if k == 0 else 5)
        Z += npnt * (side(a) + side(b)) + (nr - npnt) * (3 * (a >= 0 and bt[a] == 1) + 3 * (b >= 0 and bt[b] == 1))
        X += 2
        R += nr
        n_C += nr
    nt = int(dims["n_tets"])
    Z += nt * 3 * 12
    X += 4 * nt
    R += 3 * nt
    n_C += 9 * nt
    for a, b in contact_bodies:
        Z += 3 * (side(a) + side(b))
        X += 2
        R += 3
        n_C += 3
    D = int(dims["num_dof"])
    Dp = int(3 * np.sum(bt == 0))
    Br = int(np.sum(bt == 1))
    v = value_bytes
    return 2 * (v * Z + 4 * X) + v * n_C + 2 * v * D + v * Dp + 7 * v * Br + 13 * v * R


def cpu_baseline(args, n_env_total):
    """The reference's CPU path (oracle restatement of step_world) on the host
    cores: the same C5 envs (seeds 0..n-1), the same actions, warmed up the same
    W steps, then a bounded sample of the timed steps sized to ~cpu_seconds."""
    from oracle import oracle_py as O

    n_env = min(n_env_total, 4096)
    W = args.warmup
    t, used, _ = O.c5_bench(0, n_env, 1, not args.passive, warm=0)  # calibration
    steps = max(1, min(args.steps, int(args.cpu_seconds / max(t, 1e-3))))
    t, used, _ = O.c5_bench(0, n_env, steps, not args.passive, warm=W)
    return {"value": n_env * steps / t, "unit": "env-steps/s", "cores": used, "kind": "port",
            "sample": f"{n_env} C5 ant envs, steps {W}..{W + steps} after {W} untimed warm-up steps "
                      f"(oracle step_world, 4 Newton x 10 PCR, OpenMP over envs, {used} threads), {t:.2f} s"}


def run_reference(args):
    ws, rank, _ = dist_info()
    if rank != 0:
        return
    cb = cpu_baseline(args, args.envs)
    # each bench "step" = one bounded sample step over the workload; report the rate
    line = {"impl": "reference", "metric": "env-steps/sec at fixed Newton/CR iters", "value": cb["value"],
            "unit": "env-steps/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000.0 * args.envs / cb["value"], "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(args, ws),
            "cpu_baseline": cb, "e2e": {"value": cb["value"], "unit": "env-steps/s", "h2d_bytes_per_step": 0,
                                        "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def workload_config(args, ws):
    return {"workload": "C5 batched RL: ant environments (torso sphere + 8 box links, 8 revolute joints, "
                        "ground contact, mu=1), one step_world per env per step",
            "envs_per_gpu": args.envs, "global_envs": args.envs * ws, "newton_iterations": 4,
            "linear_iterations": 10, "linear_tolerance": 1e-10, "ncp": "fischer-burmeister",
            "r_strategy": "effective-mass", "actuated": not args.passive, "parallelism": f"env-shard x{ws}",
            "l2": "flushed (256 MiB memset) between timed steps"}


def measure(args, prec, T, tmpl, E, env0, ws, rank, local, sample_clocks):
    """Time K steps of one BatchSolver at precision `prec`: device-resident value,
    then end-to-end through the C ABI. Returns a dict of raw timings."""
    import torch

    from paper_1907_04587_b200 import BatchSolver
    from paper_1907_04587_b200.shard import action_torques, shard_states

    q0, u0 = shard_states("c5", rank, ws, E, T.num_coord, T.num_dof)
    cfg = tmpl.config
    cfg.precision = prec
    b = BatchSolver(T, tmpl.shapes, tmpl.n_shapes, tmpl.margin, tmpl.mu_default, cfg, E, args.max_contacts,
                    device=local)
    stream = torch.cuda.Stream(device=local)  # non-default stream: the C ABI reads handle 0 as "own stream"
    torch.cuda.set_stream(stream)
    b.set_stream(stream.cuda_stream)
    b.set_state(q0, u0)
    nj = T.n_joints
    K, W = args.steps, args.warmup
    # actions: a pure function of (global env id, step, joint), the same stream the CPU arm uses
    tdt = torch.float32 if prec == "fp32" else torch.float64
    torques = torch.from_numpy(action_torques(range(env0, env0 + E), range(K + W), nj)).to(tdt).cuda()
    tdt_code = 0 if prec == "fp32" else 1
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def step(i):
        ptr = None if args.passive else torques[i].data_ptr()
        b.step_device(tmpl.h, tmpl.gravity, ptr, tdt_code)

    for i in range(W):
        step(i)
    torch.cuda.synchronize()
    b.results()  # raises on contact overflow / errors
    q_w, u_w = b.get_state()  # post-warmup state: the e2e region replays the same steps

    # ---- value: device-resident inputs, L2 flushed between steps; CUDA events around
    # every step, plus (inside the library) around each of the step's launches
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    sampler = ClockSampler(local) if sample_clocks else None
    b.profile(cycles=False, launch_timing=True)
    b.counters()  # reset
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    if sampler:
        sampler.start()
        sampler.begin()
    for k in range(K):
        flush.zero_()
        ev[k][0].record(stream)
        step(W + k)
        ev[k][1].record(stream)
    torch.cuda.synchronize()
    if sampler:
        sampler.end()
    clocks = sampler.stop() if sampler else None
    if ws > 1:
        torch.distributed.barrier()
    dev_ms = sum(a.elapsed_time(bb) for a, bb in ev)
    ctr = b.counters()
    b.profile(cycles=False, launch_timing=False)
    res = b.results()  # raises if any env overflowed max_contacts in any timed step
    nc = res["n_contacts"].astype(np.float64)
    aborted = int(res["aborted"].sum())  # envs that rolled back in any timed step

    # ---- PCR-loop share of the solver's time: clock64 counters in an untimed replay
    # of the same steps (the counters' atomics stay out of the timed region)
    b.set_state(q_w, u_w)
    b.profile(cycles=True, launch_timing=False)
    b.counters()
    for k in range(min(K, 20)):
        step(W + k)
    prof = b.counters()
    b.profile(cycles=False, launch_timing=False)
    b.results()
    cr_share = prof["cr_cycles"] / prof["env_cycles"] if prof["env_cycles"] else None

    # ---- e2e: host actions -> H2D, step, D2H of the state, through the C ABI,
    # replaying the timed steps from the same post-warmup state with the same actions
    b.set_state(q_w, u_w)
    dt = torch.float64  # the batch state is fp64 in both precisions (fp32 = mixed: fp32 PCR operator)
    h_tq = torch.empty((K, E, nj), dtype=tdt, pin_memory=True)
    h_tq.copy_(torques[W:W + K].cpu())
    d_tq = torch.empty((E, nj), dtype=tdt, device="cuda")
    h_q = torch.empty((K, E * T.num_coord), dtype=dt, pin_memory=True)
    h_u = torch.empty((K, E * T.num_dof), dtype=dt, pin_memory=True)
    def e2e_run(mapped):
        # mapped (the headline): nsd_batch_step_mapped — the step kernel reads the
        # actions from, and writes the state to, the pinned host buffers itself.
        # copy: H2D copy of the actions, step_device, D2H copy of the state.
        b.set_state(q_w, u_w)
        ev2 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        for k in range(K):
            flush.zero_()
            ev2[k][0].record(stream)
            if mapped:
                b.step_mapped(tmpl.h, tmpl.gravity, None if args.passive else h_tq[k].data_ptr(), tdt_code,
                              h_q[k].data_ptr(), h_u[k].data_ptr())
            else:
                if not args.passive:
                    d_tq.copy_(h_tq[k], non_blocking=True)
                b.step_device(tmpl.h, tmpl.gravity, None if args.passive else d_tq.data_ptr(), tdt_code)
                b.copy_state_async(h_q[k].data_ptr(), h_u[k].data_ptr())
            ev2[k][1].record(stream)
        torch.cuda.synchronize()
        return sum(a.elapsed_time(bb) for a, bb in ev2)

    e2e_copy_ms = e2e_run(False)
    q_copy, u_copy = h_q[K - 1].clone(), h_u[K - 1].clone()
    e2e_ms = e2e_run(True)
    if not (torch.equal(q_copy, h_q[K - 1]) and torch.equal(u_copy, h_u[K - 1])):
        raise RuntimeError("nsd_batch_step_mapped and the copy path disagree on the final state")
    b.results()
    b.close()
    h2d = 0 if args.passive else E * nj * h_tq.element_size()
    d2h = E * (T.num_coord + T.num_dof) * 8
    if ws > 1:
        t = torch.tensor([dev_ms, e2e_ms, e2e_copy_ms], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        dev_ms, e2e_ms, e2e_copy_ms = float(t[0]), float(t[1]), float(t[2])
    total_envs = E * ws
    ns = min(E, PARITY_SAMPLE_ENVS)  # the first envs' final state, for the oracle parity sample
    q_fin = h_q[K - 1][: ns * T.num_coord].numpy().reshape(ns, T.num_coord).copy()
    u_fin = h_u[K - 1][: ns * T.num_dof].numpy().reshape(ns, T.num_dof).copy()
    return dict(dev_ms=dev_ms, e2e_ms=e2e_ms, value=total_envs * K / (dev_ms / 1000.0), q_fin=q_fin, u_fin=u_fin,
                e2e=total_envs * K / (e2e_ms / 1000.0), e2e_copy=total_envs * K / (e2e_copy_ms / 1000.0), nc=nc,
                aborted=aborted, clocks=clocks, h2d=h2d, d2h=d2h, cfg=cfg, ctr=ctr, cr_share=cr_share, E=E)


PARITY_SAMPLE_ENVS = 64


def parity_sample(args, m, env0, T, prec):
    """The bench run itself against the oracle: the first PARITY_SAMPLE_ENVS envs of
    the shard after all W + K steps (same initial states and action stream, oracle
    step_world on the host cores), max relative error of q and u over the sample.
    Stated tolerance: fp64 1e-6 (C5 tracks the oracle to ~1e-14 over 25 steps,
    tests/test_gpu_batch.py; rounding grows over 200+ contact-rich steps). fp32
    mixed mode: over 200+ actuated steps the ants' contact dynamics amplify any
    rounding chaotically, so the bound is max(1e-4, 10x the oracle's own change when
    its initial q carries fp32-sized (2^-24) relative perturbations), the rule
    tests/test_world.py states for the fp32 mode."""
    from oracle import oracle_py as O

    n = m["q_fin"].shape[0]
    steps = args.warmup + args.steps
    t0 = time.perf_counter()
    act = not args.passive
    oq, ou, onc = O.c5_states(env0, n, steps, T.num_coord, T.num_dof, actuated=act)
    rel = lambda a, b, fl: float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), fl))
    eq, eu = rel(m["q_fin"], oq, 1e-12), rel(m["u_fin"], ou, 1e-3)
    out = {"envs": n, "env_ids": f"{env0}..{env0 + n - 1}", "steps": steps, "max_rel_err_q": eq, "max_rel_err_u": eu}
    if prec == "fp64":
        tol = 1e-6
    else:
        sd = max(rel(O.c5_states(env0, n, steps, T.num_coord, T.num_dof, actuated=act, perturb=2.0 ** -24,
                                 pseed=k)[0], oq, 1e-12) for k in (1, 2))
        tol = max(1e-4, 10 * sd)
        out["oracle_self_divergence_q"] = sd
    out.update({"tolerance_q": tol, "pass": bool(eq <= tol), "oracle_seconds": time.perf_counter() - t0,
                "note": "final (q, u) of the timed run (e2e replay) vs the oracle's step_world from the same initial "
                        "states and actions"})
    return out


def traffic_record(kernel_key):
    """DRAM bytes per launch of the dominant kernel from the committed ncu capture,
    only if the kernel sources still hash to what was profiled (else null)."""
    import hashlib

    path = os.path.join(ROOT, "profiles", "dram_traffic.json")
    try:
        rec = json.load(open(path)).get(kernel_key)
        h = hashlib.sha256()
        for f in rec["sources"]:
            h.update(open(os.path.join(ROOT, f), "rb").read())
        return rec["bytes"] if h.hexdigest() == rec["sha256"] else None
    except Exception:
        return None


def roofline(m, prec, K):
    """Roofline of the dominant kernel (k_batch_warp): SURVEY §8(d) algorithmic bytes
    of the PCR iterations actually run ÷ its CUDA-event time in the timed region."""
    vb = 4 if prec == "fp32" else 8
    c = m["ctr"]
    b0 = float(b_cr_bytes(0, value_bytes=vb))
    b1 = float(b_cr_bytes(1, value_bytes=vb)) - b0  # bytes per contact
    bytes_total = b0 * c["cr_iterations"] + b1 * c["cr_iterations_x_contacts"]
    peak, peak_kind = hbm_peak()
    t_kernel = c["warp_solver_ms"] / 1000.0
    t_step = m["dev_ms"] / 1000.0
    per_launch = bytes_total / max(K, 1)
    out = {"bound": "hbm", "achieved": bytes_total / t_kernel / 1e9 if t_kernel else None, "peak": peak,
           "unit": "GB/s", "frac": None, "traffic": traffic_record(f"k_batch_warp<{'double' if vb == 8 else 'float'}>"),
           "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)" if peak_kind == "measured" else peak_kind,
           "kernel": f"k_batch_warp<{'double' if vb == 8 else 'float'}>",
           "bytes_per_launch": per_launch, "kernel_ms_per_launch": 1000.0 * t_kernel / max(K, 1),
           "pcr_iterations_per_env_step": c["cr_iterations"] / max(c["env_steps"], 1),
           "model": "SURVEY 8(d) B_CR(nc) per env per PCR iteration actually run (nsd_batch_counters), "
                    "summed over envs; kernel time from CUDA events around its launches in the timed region"}
    if out["achieved"]:
        out["frac"] = out["achieved"] / peak
    out["frac_step"] = bytes_total / t_step / 1e9 / peak
    if m["cr_share"] and t_kernel:
        t_cr = t_kernel * m["cr_share"]
        out["frac_cr_loop"] = bytes_total / t_cr / 1e9 / peak
        out["cr_loop_share_of_kernel"] = m["cr_share"]
        out["us_per_cr_iter_loop"] = 1e6 * t_cr / max(K, 1) / (c["cr_iterations"] / max(c["env_steps"], 1))
    out["launch_ms_per_step"] = {"narrow_phase": c["narrow_phase_ms"] / max(K, 1),
                                 "warp_solver": c["warp_solver_ms"] / max(K, 1),
                                 "large_envs": c["large_env_ms"] / max(K, 1)}
    return out


def scene_steps(w, steps, vb):
    """K timed World.step calls (L2 flushed before each): device ms per step from the
    CUDA events inside nsd_step (the step is ONE kernel launch), wall seconds, PCR
    iterations run, and the SURVEY §8(d) bytes of those iterations (B_CR from the
    step's exact structure and contact set)."""
    import torch

    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    dev, wall, pcr, nbytes, ncs = [], [], 0, 0.0, []
    for _ in range(steps):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rep = w.step()
        wall.append(time.perf_counter() - t0)
        dev.append(rep["ms"])
        it = int(sum(rep["stats"][:, 5]))
        pcr += it
        ib = w.contacts[0] if w.contacts is not None else np.zeros((0, 3), np.int32)
        ncs.append(len(ib))
        nbytes += it * scene_b_cr(w.scene.dims, w.topology, len(ib), [(int(a), int(b)) for a, b in ib[:, :2]], vb)
    return dev, wall, pcr, nbytes, ncs


def scene_roofline(dev, nbytes):
    peak, kind = hbm_peak()
    t = sum(dev) / 1000.0
    ach = nbytes / t / 1e9 if t else None
    return {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak if ach else None,
            "traffic": None, "peak_source": kind, "bytes_per_launch": nbytes / max(len(dev), 1),
            "model": "SURVEY 8(d) B_CR of the step's structure x PCR iterations run, over the nsd_step kernel's "
                     "CUDA-event time (the whole step: assembly, SVD/eigen per tet and PCR in one launch)"}


def scene_summary(name, precision, steps, warmup):
    """ms/step and us per CR iteration of one single scene through World.step
    (device time per step from CUDA events in nsd_step, L2 flushed between steps)."""
    import torch

    from paper_1907_04587_b200 import World

    w = World(name, 0, precision=precision)
    for _ in range(warmup):
        w.step()
    dev, wall, pcr, nbytes, ncs = scene_steps(w, steps, 4 if precision == "fp32" else 8)
    cfg = w.config
    ms = float(np.mean(dev))
    out = {"ms_per_step": ms, "us_per_cr_iter_budget": 1000.0 * ms / (cfg.newton_iterations * cfg.linear_max_iterations),
           "us_per_cr_iter_used": 1000.0 * ms * steps / max(pcr, 1), "pcr_iterations_per_step": pcr / steps,
           "steps_per_s": 1000.0 / ms, "e2e_steps_per_s": 1.0 / float(np.mean(wall)),
           "budget": f"{cfg.newton_iterations}x{cfg.linear_max_iterations}", "tets": w.scene.dims["n_tets"],
           "bodies": w.scene.dims["n_bodies"], "mean_contacts": float(np.mean(ncs)),
           "roofline": scene_roofline(dev, nbytes)}
    w.close()
    return out


def run_scene(args):
    """One scene per GPU (C1-C4 are replicas only): K x step_world through
    the public World API. value = steps/s from the device time of each step's kernel
    (CUDA events inside nsd_step), L2 flushed between steps; e2e = wall clock of
    World.step (host detect + H2D + kernel + D2H)."""
    import torch

    from paper_1907_04587_b200 import World

    ws, rank, local = dist_info()
    torch.cuda.set_device(local)
    K, W = args.steps, args.warmup
    w = World(args.workload, 0, precision=args.precision)
    for _ in range(W):
        w.step()
    sampler = ClockSampler(local)
    sampler.start()
    sampler.begin()
    dev, wall, pcr, nbytes, ncs = scene_steps(w, K, 4 if args.precision == "fp32" else 8)
    clocks = sampler.stop()
    cfg = w.config
    ms = float(np.mean(dev))
    cr_budget = cfg.newton_iterations * cfg.linear_max_iterations
    cpu = None
    if not args.no_cpu_baseline:
        from oracle import oracle_py as O

        ow = O.OracleWorld(args.workload, 0)
        ow.step(W)
        n = 0
        t0 = time.perf_counter()
        while n < K and time.perf_counter() - t0 < args.cpu_seconds:
            ow.step(1)
            n += 1
        t = time.perf_counter() - t0
        cpu = {"value": n / t, "unit": "steps/s", "cores": os.cpu_count(), "kind": "port",
               "sample": f"{args.workload}: oracle step_world steps {W}..{W + n} ({t:.2f} s)"}
    line = {"metric": "steps/sec at fixed Newton/CR iters (single scene)", "value": 1000.0 / ms, "unit": "steps/s",
            "n_gpus": ws, "steps": K, "warmup": W, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32" if args.precision == "fp32" else "f64", "data": "synthetic",
            "config": {"workload": args.workload, "bodies": w.scene.dims["n_bodies"], "tets": w.scene.dims["n_tets"],
                       "newton_iterations": cfg.newton_iterations, "linear_iterations": cfg.linear_max_iterations,
                       "parallelism": "replicas only", "l2": "flushed (256 MiB memset) between timed steps"},
            "us_per_cr_iter_budget": 1000.0 * ms / cr_budget, "pcr_iterations_used_per_step": pcr / K,
            "us_per_cr_iter_used": 1000.0 * ms * K / max(pcr, 1), "mean_contacts": float(np.mean(ncs)),
            "roofline": scene_roofline(dev, nbytes),
            "e2e": {"value": 1.0 / float(np.mean(wall)), "unit": "steps/s",
                    "h2d_bytes_per_step": 8 * (w.scene.dims["num_coord"] + w.scene.dims["num_dof"]),
                    "d2h_bytes_per_step": 8 * (w.scene.dims["num_coord"] + w.scene.dims["num_dof"])},
            "gpu_launches": K, "clocks": clocks}
    if cpu:
        line["cpu_baseline"] = cpu
    print(json.dumps(line), flush=True)
    w.close()


def main():
    args = parse()
    maybe_relaunch(args)
    if args.impl == "reference":
        run_reference(args)
        return
    if args.workload != "c5":
        run_scene(args)
        return
    import torch

    ws, rank, local = dist_info()
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1907_04587_b200 import Scene

    if args.team:
        os.environ["NSD_BATCH_TEAM"] = str(args.team)
    from paper_1907_04587_b200.shard import env_range

    env0, E = env_range(rank, ws, args.envs)
    tmpl = Scene("c5", env0)
    T = tmpl.topology
    K, W = args.steps, args.warmup
    prec = args.precision
    m = measure(args, prec, T, tmpl, E, env0, ws, rank, local, True)
    other = None
    if not args.no_alt:
        alt = "fp32" if prec == "fp64" else "fp64"
        a = measure(args, alt, T, tmpl, E, env0, ws, rank, local, False)
        other = {"dtype": "f32" if alt == "fp32" else "f64", "value": a["value"], "ms_per_step": a["dev_ms"] / K,
                 "e2e": a["e2e"], "e2e_copy_path": a["e2e_copy"], "roofline_frac": roofline(a, alt, K)["frac"],
                 "mode": ("mixed precision: fp64 state, assembly, Newton update and reductions; fp32 PCR operator "
                          "and row vectors") if alt == "fp32" else "fp64",
                 "parity": ("oracle parity 1e-4 over 25 steps (tests/test_gpu_batch.py)") if alt == "fp32"
                 else "oracle parity 1e-8 over 25 steps"}
        if not args.no_parity_sample and rank == 0:
            try:
                other["parity_sample"] = parity_sample(args, a, env0, T, alt)
            except Exception as e:  # reported, never fatal
                other["parity_sample"] = {"error": str(e)}
    if rank != 0:
        if ws > 1:
            torch.distributed.destroy_process_group()
        return
    cfg = m["cfg"]
    line = {"metric": "env-steps/sec at fixed Newton/CR iters", "value": m["value"], "unit": "env-steps/s",
            "n_gpus": ws, "steps": K, "warmup": W, "ms_per_step": m["dev_ms"] / K, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32" if prec == "fp32" else "f64",
            "data": "synthetic", "config": workload_config(args, ws),
            "us_per_cr_iter": 1000.0 * (m["dev_ms"] / K) / (m["ctr"]["cr_iterations"] / max(m["ctr"]["env_steps"], 1)),
            "us_per_cr_iter_note": "whole step (3 launches) per PCR iteration run per env-step; "
                                   "roofline.us_per_cr_iter_loop is the PCR loops alone",
            "mean_contacts_per_env": float(m["nc"].mean()), "aborted_envs": m["aborted"],
            "roofline": roofline(m, prec, K),
            "e2e": {"value": m["e2e"], "unit": "env-steps/s", "h2d_bytes_per_step": m["h2d"],
                    "d2h_bytes_per_step": m["d2h"],
                    "path": "nsd_batch_step_mapped: the step kernel reads the actions from and writes (q, u) to "
                            "pinned host memory",
                    "copy_path_value": m["e2e_copy"]},
            "gpu_launches": 3 * K, "clocks": m["clocks"]}
    if other:
        line["other_precision"] = other
    if not args.no_parity_sample:
        try:
            line["parity_sample"] = parity_sample(args, m, env0, T, prec)
        except Exception as e:  # reported, never fatal for the headline
            line["parity_sample"] = {"error": str(e)}
    if ws == 1 and not args.no_scenes:
        # the other BASELINE configs (single scenes, replicas only), fp64, 20 steps each
        line["single_scenes"] = {}
        for name in ("c1", "c3", "c2", "c4"):
            try:
                line["single_scenes"][name] = scene_summary(name, "fp64", 20, 3)
            except Exception as e:  # reported, never fatal for the headline
                line["single_scenes"][name] = {"error": str(e)}
    if ws == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline(args, E)
        except Exception as e:  # the baseline is reported, never required
            line["cpu_baseline"] = {"value": None, "error": str(e)}
    print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
