"""The reference's JSON scene format (parse_scene / serialize_scene, scene.h:74-77,
src/scene.cpp:1-556) on the product's scene layer (csrc/nsd_scene_json.cpp).

* Round trip: serialize_scene of every builder scene the format can carry, parsed
  back, builds the same world (topology, shapes, config bit for bit; orientations
  to one rounding of the reference's renormalisation) and serializes to the same
  text.
* Layout: nlohmann::json (the reference's JSON library; test-side tool
  tests/cpp/json_dump_ref.cpp, skipped when its header is not in the image) reads
  the text as the same document and its dump(2) has the same layout token for
  token. Numbers are compared by value: the product prints the shortest
  round-trip digits, nlohmann's Grisu2 occasionally a longer spelling of the same
  double. The image's copy (cudnn_frontend's) also prints integer arrays on one
  line, a local patch to the stock serializer, so mesh element arrays are compared
  as values only.
* Validation: the reference's rules and messages for rejected documents.
* The C++ API: world_from_json / serialize_scene (include/nsdyn_b200.hpp).
"""
import glob
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

ROUNDTRIP = ["box_on_plane", "heavy_stack", "arch", "box_pile", "incline:35:0.5", "stretch_sheet",
             "stretch_sheet_linear", "c1", "c3:30", "c5"]


def _scene(name=None, text=None):
    from paper_1907_04587_b200 import Scene

    return Scene(name) if text is None else Scene.from_json(text)


def _same_world(a, b):
    ta, tb = a.topology, b.topology
    for f in ("body_type", "body_mass", "body_inertia", "joint_kind", "joint_body", "joint_frame", "joint_param",
              "tet_body", "tet_dm_inv", "tet_volume", "tet_material"):
        assert np.array_equal(ta.a[f], tb.a[f]), f
    assert a.dims == b.dims
    assert np.array_equal(a.u, b.u)
    assert np.max(np.abs(a.q - b.q), initial=0.0) <= 1e-15  # renormalised orientations (bodies.cpp:52-56)
    for x, y in zip(a.shapes[:a.n_shapes], b.shapes[:b.n_shapes]):  # normals renormalised on parse (scene.cpp)
        assert (x.body, x.kind, x.offset, x.radius, x.thickness, x.mu) == (y.body, y.kind, y.offset, y.radius,
                                                                          y.thickness, y.mu)
        assert list(x.half_extents) == list(y.half_extents)
        assert np.max(np.abs(np.array(x.normal) - np.array(y.normal))) <= 1e-15
    assert (a.margin, a.mu_default, a.h) == (b.margin, b.mu_default, b.h)
    assert np.array_equal(a.gravity, b.gravity)
    assert vars(a.config) == vars(b.config)


def _same_doc(a, b, tol_key=None, path="$"):
    """Exact equality of two parsed documents (ints stay ints); values under
    a key in `tol_key` (orientation, half-space normal) to 1e-15."""
    assert type(a) is type(b), path
    if isinstance(a, dict):
        assert a.keys() == b.keys(), path
        for k in a:
            _same_doc(a[k], b[k], tol_key, path + "." + k)
    elif isinstance(a, list):
        assert len(a) == len(b), path
        for i, (x, y) in enumerate(zip(a, b)):
            _same_doc(x, y, tol_key, f"{path}[{i}]")
    elif tol_key and any(k in path for k in tol_key) and isinstance(a, float):
        assert abs(a - b) <= 1e-15, path
    else:
        assert a == b, path


@pytest.mark.parametrize("name", ROUNDTRIP)
def test_roundtrip_builds_the_same_world(name):
    """The reference renormalises [w,x,y,z] and half-space normals on parse
    (bodies.cpp:52-56, scene.cpp parse_shape), so those may move by one rounding per
    round trip; everything else is exact."""
    import json

    s = _scene(name)
    text = s.to_json()
    r = _scene(text=text)
    _same_world(s, r)
    _same_doc(json.loads(text), json.loads(r.to_json()), tol_key=("orientation", "normal"))


def _nlohmann_dump():
    hdrs = glob.glob(os.path.join(sys.prefix, "lib", "python*", "site-packages", "**", "nlohmann", "json.hpp"),
                     recursive=True)
    if not hdrs:
        pytest.skip("nlohmann/json.hpp not in this image")
    inc = os.path.dirname(os.path.dirname(hdrs[0]))
    out = os.path.join(ROOT, "tests", "cpp", "_build", "json_dump_ref")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    src = os.path.join(ROOT, "tests", "cpp", "json_dump_ref.cpp")
    if not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(src):
        r = subprocess.run(["g++", "-std=c++17", "-O1", "-I", inc, src, "-o", out], capture_output=True, text=True)
        if r.returncode != 0:
            pytest.skip("nlohmann tool does not build: " + r.stderr[-300:])
    return lambda text: subprocess.run([out], input=text, capture_output=True, text=True, check=True).stdout


def _tokens(text, compact_int_arrays=False):
    """Layout tokens with numbers as values; optionally integer arrays collapsed."""
    import re

    if compact_int_arrays:
        text = re.sub(r"\[\s*(-?\d+(?:\s*,\s*-?\d+)*)\s*\]", lambda m: "[" + re.sub(r"\s+", "", m.group(1)) + "]", text)
    out = []
    for m in re.finditer(r"-?\d+(?:\.\d+)?(?:[eE][+-]?\d+)?|\s+|.", text):
        t = m.group(0)
        if t[0].isdigit() or (t[0] == "-" and len(t) > 1):
            out.append(float(t) if any(c in t for c in ".eE") else int(t))
        else:
            out.append(t)
    return out


@pytest.mark.parametrize("name", ["c1", "c5", "box_pile", "stretch_sheet", "incline:35:0.5", "arch"])
def test_layout_matches_nlohmann_dump(name):
    import json

    dump = _nlohmann_dump()
    text = _scene(name).to_json()
    ref = dump(text)
    _same_doc(json.loads(ref), json.loads(text))
    assert _tokens(ref, True) == _tokens(text, True)


def test_number_layout_matches_nlohmann():
    """Edge values of the float layout (shortest round trip, '.0', exponent range)."""
    dump = _nlohmann_dump()
    vals = [0.0, -0.0, 1.0, -9.81, 0.0083, 1e-10, 1e-5, 1e-4, 0.001, 123456789012345.0, 1e15, 1e16, 1.5e-7, 2.0 / 3.0,
            1e300, 5e-324, 0.1 + 0.2, 1234.5678, -1e-300, 7e22]
    body = ",\n".join(f"  {v!r}" if v != 0 else ("  -0.0" if str(v).startswith("-") else "  0.0") for v in vals)
    doc = "{\n  \"timestep\": 0.5,\n  \"gravity\": [0.0, 0.0, -9.81]\n}\n"
    from paper_1907_04587_b200 import Scene

    # through the product serializer: every value as a mass of a particle body
    bodies = ",".join(f'{{"type": "particle", "mass": {abs(v) if v != 0 else 1.0!r}, "position": [{v!r}, 0, 0]}}'
                      for v in vals)
    text = Scene.from_json('{"bodies": [' + bodies + ']}').to_json()
    assert _tokens(dump(text)) == _tokens(text)
    assert doc and body  # layout inputs built above


def test_defaults_and_orientation_forms():
    s = _scene(text='{"bodies": [{"type": "rigid", "mass": 2, "shape": {"kind": "sphere", "radius": 0.5},'
                    ' "orientation": {"axis": [0, 0, 2], "angle_deg": 90}},'
                    ' {"type": "rigid", "mass": 1, "shape": {"kind": "box", "half_extents": [1, 1, 1]},'
                    ' "orientation": [2, 0, 0, 0]}]}')
    assert s.h == 0.0083 and list(s.gravity) == [0.0, 0.0, -9.81]
    assert (s.margin, s.mu_default) == (0.01, 0.5)
    c = s.config
    assert (c.newton_iterations, c.linear_max_iterations, c.linear_tolerance, c.step_fraction) == (8, 40, 1e-10, 0.75)
    q = s.q
    h = np.sqrt(0.5)
    assert np.allclose(q[3:7], [h, 0, 0, h], atol=1e-15)
    assert np.array_equal(q[10:14], [1.0, 0.0, 0.0, 0.0])


ERRORS = [
    ('{"foo": 1}', 'scene error at $: unknown key "foo"'),
    ("[1, 2]", "scene error at $: expected an object"),
    ('{"timestep": 0}', "scene error at $.timestep: must be positive"),
    ('{"bodies": [{"type": "rigid", "mass": -1, "shape": {"kind": "sphere", "radius": 1}}]}',
     "scene error at bodies[0].mass: must be positive"),
    ('{"bodies": [{"type": "rigid", "mass": 1}]}',
     "scene error at bodies[0]: rigid body needs a shape or an explicit inertia"),
    ('{"bodies": [{"type": "rigid", "mass": 1, "shape": {"kind": "halfspace"}}]}',
     "scene error at bodies[0].shape: half-spaces must be static bodies"),
    ('{"bodies": [{"type": "static"}]}', "scene error at bodies[0].shape: missing"),
    ('{"bodies": [{"type": "ghost"}]}', 'scene error at bodies[0].type: unknown body type "ghost"'),
    ('{"bodies": [{"type": "rigid", "mass": 1, "shape": {"kind": "box", "half_extents": [1, 0, 1]}}]}',
     "scene error at bodies[0].shape.half_extents: must be positive"),
    ('{"bodies": [{"type": "particle", "mass": 1, "position": [0, 0]}]}',
     "scene error at bodies[0].position: expected an array of 3 numbers"),
    ('{"bodies": [{"type": "rigid", "mass": 1, "inertia": [[1, 0, 0], [0, 1, 0]]}]}',
     "scene error at bodies[0].inertia: expected a 3x3 matrix"),
    ('{"bodies": [{"type": "static", "shape": {"kind": "halfspace"}}], "joints": [{"type": "fixed_point", "body_a": 0}]}',
     "scene error at joints[0]: joints cannot attach to static bodies; use body -1 for the world"),
    ('{"joints": [{"type": "fixed_point", "body_a": 3}]}', "scene error at joints[0]: body index out of range"),
    ('{"joints": [{"type": "bend_spring"}]}', "scene error at joints[0].stiffness: bend springs need a positive stiffness"),
    ('{"joints": [{"type": "hinge"}]}', 'scene error at joints[0].type: unknown joint type "hinge"'),
    ('{"joints": [{"type": "revolute", "axis": [0, 0, 0]}]}', "scene error at joints[0].axis: zero-length axis"),
    ('{"meshes": [{"vertices": [[0, 0, 0]], "elements": [[0, 0, 0, 1]], "material": {"model": "linear", "young": 1, "poisson": 0.3}}]}',
     "scene error at meshes[0].elements[0]: vertex index out of range"),
    ('{"meshes": [{"vertices": [], "elements": [], "material": {"model": "neohookean", "young": 1, "poisson": 0.5}}]}',
     "scene error at meshes[0].material.poisson: must lie in [0, 0.4999)"),
    ('{"meshes": [{"vertices": [], "elements": []}]}', "scene error at meshes[0].material: missing"),
    ('{"solver": {"linear": {"iterations": 5}}}', "scene error at $.solver.linear.method: missing"),
    ('{"solver": {"linear": {"method": "pcr", "iterations": 5.0}}}',
     "scene error at $.solver.linear.iterations: expected an integer"),
    ('{"solver": {"step_fraction": 1.5}}', "scene error at $.solver.step_fraction: must lie in (0, 1]"),
    ('{"solver": {"ncp": "abs"}}', 'scene error at $.solver.ncp: unknown NCP function "abs"'),
    ('{"solver": {"r_strategy": "mass"}}', 'scene error at $.solver.r_strategy: unknown strategy "mass"'),
    ('{"contacts": {"margin": -1}}', "scene error at $.contacts.margin: must be >= 0"),
    ('{"bodies": [{"type": "rigid", "mass": 1, "shape": {"kind": "sphere", "radius": 1}, "orientation": [1, 0, 0]}]}',
     "scene error at bodies[0].orientation: expected a quaternion [w,x,y,z]"),
]


@pytest.mark.parametrize("doc,msg", ERRORS)
def test_validation_messages(doc, msg):
    from paper_1907_04587_b200 import NsdError

    with pytest.raises(NsdError) as e:
        _scene(text=doc)
    assert str(e.value).endswith(msg)


@pytest.mark.parametrize("doc", ['{"bodies": [', '{"a" 1}', '{"timestep": 01}', '{"x": tru}', ""])
def test_syntax_errors(doc):
    from paper_1907_04587_b200 import NsdError

    with pytest.raises(NsdError) as e:
        _scene(text=doc)
    assert "scene syntax error: " in str(e.value)


def test_cpp_api_json_roundtrip_and_errors(tmp_path):
    exe = os.path.join(ROOT, "tests", "cpp", "_build", "world_demo")
    r = subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    for name in ("c1", "c5", "stretch_sheet"):
        r = subprocess.run([exe, "--json-roundtrip", name], capture_output=True, text=True)
        assert r.returncode == 0 and r.stdout.endswith("json_roundtrip ok\n"), r.stdout[-300:] + r.stderr
        assert r.stdout[: -len("json_roundtrip ok\n")] == _scene(name).to_json()
    bad = tmp_path / "bad.json"
    bad.write_text('{"bodies": [{"type": "particle", "mass": 0}]}')
    r = subprocess.run([exe, "--json-load", str(bad)], capture_output=True, text=True)
    assert r.returncode == 1 and "json_error scene error at bodies[0].mass: must be positive" in r.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c1", "c5"])
def test_json_scene_steps_like_the_builder(name, tmp_path):
    """A scene loaded from its JSON document steps bit for bit like the builder
    scene: through the Python World and through the C++ runner given the file
    (load_world, runner.cpp:130-146)."""
    from paper_1907_04587_b200 import World

    text = _scene(name).to_json()
    a, b = World(name, 0, precision="fp64"), World(json_text=text, precision="fp64")
    exact = np.array_equal(a.q, b.q)  # False when an orientation was renormalised by one rounding
    for _ in range(5):
        a.step(1)
        b.step(1)
    if exact:
        assert np.array_equal(a.q, b.q) and np.array_equal(a.u, b.u)
    else:
        assert np.max(np.abs(a.q - b.q)) < 1e-12 and np.max(np.abs(a.u - b.u)) < 1e-10
    a.close()
    b.close()
    exe = os.path.join(ROOT, "tests", "cpp", "_build", "world_demo")
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)
    f = tmp_path / "scene.json"
    f.write_text(text)
    outs = []
    for scene in (name, str(f)):
        out = tmp_path / ("o_" + str(len(outs)))
        r = subprocess.run([exe, "--run", scene, "5", str(out)], capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stdout + r.stderr
        outs.append((out / "trajectory.csv").read_text())
    if exact:
        assert outs[0] == outs[1]
    else:
        ta = np.loadtxt(outs[0].splitlines()[1:], delimiter=",")
        tb = np.loadtxt(outs[1].splitlines()[1:], delimiter=",")
        assert np.max(np.abs(ta - tb)) < 1e-10
