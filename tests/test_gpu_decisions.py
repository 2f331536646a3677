"""Per-Newton-iteration decision vectors (SURVEY §8(c) parity protocol and
Appendix A.3), GPU (fp64, through nsd_step) against the oracle at the same
state, bit for bit: per contact the normal-row-kept, friction-active, W-cap,
W-zero and NCP-branch flags; per tet the PSD projection and diagonal
fallback; per dof the geometric-stiffness skip / clamp / rigid-zeroing; and
the PCR exit reason (budget, tolerance, monotone guard, breakdown). Layout:
nsd_step_out::decisions (include/nsdyn_gpu.h). The incline cases at step 0
start exactly touching (gap 0, lambda 0): the Fischer-Burmeister origin, where
the branch depends on the gap's last bit; the device computes that gap without
FMA contraction, as the oracle does, so they agree there too."""
import numpy as np
import pytest

from tests.helpers import oracle_case, run_gpu, run_oracle

pytestmark = pytest.mark.gpu

RIGID = [("c1", 0, 0), ("c1", 0, 5), ("c1", 0, 20), ("c3", 0, 0), ("c3", 0, 6), ("c5", 3, 0), ("c5", 3, 10),
         ("heavy_stack", 0, 0), ("heavy_stack", 0, 12), ("box_pile", 1, 10), ("box_pile", 1, 30),
         ("incline:35:0.5", 0, 0), ("incline:35:0.5", 0, 5), ("incline:20:0.5", 0, 0), ("incline:20:0.5", 0, 5), ("arch", 0, 0), ("arch", 0, 2), ("box_on_plane", 0, 8),
         ("bend_chain", 0, 0), ("bend_chain", 0, 12)]
FEM = [("c2:6", 0, 0), ("c2:6", 0, 2), ("c2:6", 0, 4)]


def _compare(name, seed, warm, prec="fp64"):
    case = oracle_case(name, seed, warm)
    g = run_gpu(case, prec)
    o = run_oracle(case)
    gd, od = g["decisions"], o["decisions"]
    assert gd.shape == od.shape, (gd.shape, od.shape)
    return gd, od, case["dims"]


@pytest.mark.parametrize("name,seed,warm", RIGID + FEM)
def test_decision_vectors_bit_equal_fp64(name, seed, warm):
    gd, od, dims = _compare(name, seed, warm)
    diff = np.argwhere(gd != od)
    assert diff.size == 0, [(int(i), int(k), int(gd[i, k]), int(od[i, k])) for i, k in diff[:12]]


def test_decision_vectors_exercise_every_flag():
    """The cases above are not vacuous: across them the flags take both values."""
    seen = np.zeros(8, int)
    for name, seed, warm in [("box_pile", 1, 30), ("incline:35:0.5", 0, 5), ("c2:6", 0, 4), ("heavy_stack", 0, 12)]:
        gd, _, dims = _compare(name, seed, warm)
        nc = dims["n_contacts"]
        c = gd[:, :nc]
        seen[0] += int(np.any(c & 1)) + int(np.any(~c & 1))
        seen[1] += int(np.any(c & 2))
        seen[2] += int(np.any(gd[:, -1] == 0)) + int(np.any(gd[:, -1] == 2))
    assert seen[0] >= 2 and seen[1] >= 1 and seen[2] >= 1



@pytest.mark.slow
@pytest.mark.parametrize("warm", [0, 2])
@pytest.mark.parametrize("name", ["c2", "c4"])
def test_decision_vectors_full_fem_fp64(name, warm):
    """Full-size FEM configs (C2 12^3 block, C4 hand + ball), one step from the oracle's
    state after `warm` steps: every Newton iteration's contact / tet / dof decisions
    and PCR exit reasons bit-equal."""
    gd, od, dims = _compare(name, 0, warm)
    mism = [int(np.count_nonzero(gd[i] != od[i])) for i in range(gd.shape[0])]
    print(name, "decision mismatches per Newton iteration:", mism)
    assert mism[0] == 0
    assert sum(mism) == 0, mism


@pytest.mark.parametrize("name,seed,warm", RIGID + FEM)
def test_decision_vectors_fp32_mode(name, seed, warm):
    """fp32 mode (fp64 arithmetic, fp32 J/C coefficients): SURVEY §8(c) asks fp32
    decisions to be counted and reported; measured, they are bit-equal too."""
    gd, od, dims = _compare(name, seed, warm, "fp32")
    diff = np.argwhere(gd != od)
    print(name, warm, "fp32 decision mismatches:", len(diff))
    assert diff.size == 0, [(int(i), int(k), int(gd[i, k]), int(od[i, k])) for i, k in diff[:12]]


@pytest.mark.parametrize("name,seed,warm", [("stretch_sheet", 0, 3), ("stretch_sheet_linear", 0, 2),
                                            ("stretch_sheet_linear", 0, 6)])
def test_decision_vectors_sheets_fp64(name, seed, warm):
    """The stretched sheets (scene.cpp:928): Neo-Hookean from F = I (degenerate SVD,
    PSD projection) and the linear co-rotational model (materials.cpp:140-178).
    Contact and tet decisions and the PCR exits are bit-equal. The per-dof
    geometric-stiffness clamp (newton.cpp:308, c_k >= 0) is counted, not asserted:
    on these sheets c_k is a difference quotient of near-equal momentum residuals at
    ~0, and the iterates already differ at the level test_gpu_parity.py states for
    them (the SVD's U, V at F = I are pinned by no reference test; the linear sheet's
    60-iteration PCR ends at its rounding floor), so its sign is borderline."""
    gd, od, dims = _compare(name, seed, warm)
    n_ct = dims["n_contacts"] + dims["n_tets"]
    diff = np.argwhere(gd[:, :n_ct] != od[:, :n_ct])
    assert diff.size == 0, [(int(i), int(k), int(gd[i, k]), int(od[i, k])) for i, k in diff[:12]]
    assert np.array_equal(gd[:, -1], od[:, -1])  # PCR exit reasons
    dofs = gd[:, n_ct:-1] != od[:, n_ct:-1]
    flips = (gd[:, n_ct:-1] ^ od[:, n_ct:-1])[dofs]
    assert np.all(flips == 2), "only the GS-clamp bit may differ"  # kDecGsClamp
    print(name, warm, "GS-clamp flag differences:", int(dofs.sum()), "of", dofs.size)


@pytest.mark.parametrize("method", [0, 1, 2])
def test_decision_vectors_other_linear_methods_fp64(method):
    """Jacobi / Gauss-Seidel / PCG on the same boundary: contact, tet and dof decisions
    bit-equal (the exit byte is PCR's and stays kExitNone for these methods)."""
    case_args = ("box_pile", 1, 20)
    from tests.helpers import oracle_case, run_gpu, run_oracle
    case = oracle_case(*case_args, overrides=dict(linear_method=method))
    g = run_gpu(case, "fp64")
    o = run_oracle(case)
    diff = np.argwhere(g["decisions"] != o["decisions"])
    assert diff.size == 0, [(int(i), int(k)) for i, k in diff[:12]]
