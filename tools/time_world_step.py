"""Host-side breakdown of World.step for one single scene (diagnostic, GPU box).
usage: python tools/time_world_step.py c4 [steps]"""
import sys
import time

import numpy as np

import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1907_04587_b200 import World, lib, check  # noqa: E402

os.environ.setdefault("NSD_HOST_TIMING", "1")
name = sys.argv[1] if len(sys.argv) > 1 else "c4"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 20
w = World(name, 0)
w.step(3)
acc = {"anchors": [], "detect": [], "newton_step": [], "device_ms": []}
for _ in range(K):
    t0 = time.perf_counter()
    check(lib().nsd_scene_advance_anchors(w._h))
    t1 = time.perf_counter()
    w.contacts = w.detect()
    t2 = time.perf_counter()
    rep = w.solver.newton_step(w.q, w.u, w.contacts, h=w.h, gravity=tuple(w.gravity), f_extra=w.f_extra,
                               joint_frame=w.joint_frames(), decisions=False)
    t3 = time.perf_counter()
    w.q, w.u = rep["q"], rep["u"]
    w.contacts = rep.get("contacts", w.contacts)
    acc["anchors"].append(1e3 * (t1 - t0))
    acc["detect"].append(1e3 * (t2 - t1))
    acc["newton_step"].append(1e3 * (t3 - t2))
    acc["device_ms"].append(rep["ms"])
print(name, {k: round(float(np.median(v)), 3) for k, v in acc.items()}, "contacts", len(w.contacts[0]))
w.close()  # prints the NSD_HOST_TIMING per-phase wall times
