"""CPU: the C-ABI library loads and exports every symbol include/gridcast_b200.h declares;
host-side logic (RNG keys through the ABI, Q recognition, factorisation, windows)."""

import json
import os
import re
import subprocess

import numpy as np
import pytest

import golden_io

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_2603_01122_b200 import _lib, build
    build.build()
    return _lib.lib()


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "gridcast_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:[\w\s\*]+?)\b(gc_\w+)\s*\(", src, flags=re.M)))


def test_header_symbols_exported(L):
    syms = declared_symbols()
    assert len(syms) >= 12, syms
    from paper_2603_01122_b200 import _lib
    assert set(syms) == set(_lib.EXPORTS)
    for s in syms:
        assert hasattr(L, s), s
    so = os.path.join(ROOT, "paper_2603_01122_b200", "_lib", "libgridcast_b200.so")
    nm = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True).stdout
    for s in syms:
        assert re.search(rf"\bT {s}$", nm, flags=re.M), s


def test_library_is_sm100a(L):
    so = os.path.join(ROOT, "paper_2603_01122_b200", "_lib", "libgridcast_b200.so")
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_reference_kernels_have_no_contracted_beta_products(L):
    """The reference-arithmetic kernels (k_predict<0, ...>) compute fl(fl(beta Q') - M) with two
    roundings; ptxas can fold a packed product into the following add as one FFMA2 with a
    scalar multiplier and a negated scalar addend (seen when the product had no other use).
    No such FFMA2 may appear in their SASS (the GPU bit-exact tests are the final guard)."""
    so = os.path.join(ROOT, "paper_2603_01122_b200", "_lib", "libgridcast_b200.so")
    sass = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s*Function : ", sass)
    ref = [f for f in funcs if re.match(r"_ZN2gc9k_predictILi0E", f)]
    assert len(ref) >= 6, len(ref)  # K = 1 / 2 / 4, two histogram paths
    pat = re.compile(r"FFMA2 R\d+, R\d+\.F32x2\.HI_LO, R\d+\.F32, -R\d+\.F32 ")
    for f in ref:
        assert not pat.search(f), f.splitlines()[0]


def test_abi_version(L):
    assert L.gc_abi_version() == 3


def test_header_constants_match_the_python_mirror():
    """Every GC_* integer constant the Python mirror restates equals the header's #define
    (status codes, error bits, RNG modes, size limits...)."""
    from paper_2603_01122_b200 import _lib
    src = open(os.path.join(ROOT, "include", "gridcast_b200.h")).read()
    defs = dict(re.findall(r"^#define (GC_\w+) \(?([0-9u <]+)\)?\s*(?:/\*.*)?$", src, flags=re.M))
    checked = 0
    for name, expr in defs.items():
        if hasattr(_lib, name):
            val = eval(expr.replace("u", ""))  # noqa: S307 -- literal ints and shifts only
            assert getattr(_lib, name) == val, (name, getattr(_lib, name), val)
            checked += 1
    assert checked >= 8, checked
    assert {"GC_MAX_HYPOTHESES", "GC_MAX_ACTIONS", "GC_MAX_SMOOTH_RADIUS"} <= set(defs)


def test_abi_rng_matches_reference_streams(L):
    from paper_2603_01122_b200 import rng
    z = golden_io.load("philox.npz")
    meta = json.loads(str(z["meta"]))
    for i, (seed, path) in enumerate(zip(meta["seeds"], meta["paths"])):
        assert rng.derive_seed(seed, *path) == int(meta["derived"][i])
        np.testing.assert_array_equal(rng.stream_f32(seed, path, 24), z["f32"][i])


def test_q_recognition():
    import paper_2603_01122_b200 as G
    from paper_2603_01122_b200.tables import recognise_q
    cs = G.ControlSet.grid(4, 24, 1.4)
    lq = recognise_q(G.q_goal_progress(0.3, (0.1, 0.2)))
    assert (lq.family, lq.tau, lq.w_v, lq.w_th, lq.full) == ("goal_progress", 0.3, 0.1, 0.2, False)
    lq = recognise_q(G.mask_stationary(G.q_goal_progress(0.5), cs, 0.5))
    assert lq.family == "goal_progress" and lq.full
    assert recognise_q(G.q_default((2.0, 3.0))).family == "default"
    assert recognise_q(G.QFunction(base=lambda xy, g, v, th: np.zeros((len(xy), len(v))))) is None


def test_q_recognition_of_reference_style_closures():
    """QFunctions built by the reference (closures named q_goal_progress.<locals>...)."""
    from paper_2603_01122_b200.tables import recognise_q

    def q_goal_progress(lookahead_s=0.5, weights=(0.0, 0.0)):
        tau = float(lookahead_s)
        w_v, w_th = float(weights[0]), float(weights[1])

        def shift_free(xy, goal_xy, v, theta):
            return tau + w_v + w_th

        def base(xy, goal_xy, v, theta):
            return shift_free(xy, goal_xy, v, theta)

        class Q:
            pass
        q = Q()
        q.base, q.base_policy, q.mask = base, shift_free, None
        return q

    lq = recognise_q(q_goal_progress(0.7, (0.5, 0.25)))
    assert (lq.tau, lq.w_v, lq.w_th, lq.full) == (0.7, 0.5, 0.25, False)
    q = q_goal_progress(0.7)
    q.base_policy = None
    lq = recognise_q(q)
    assert lq.tau == 0.7 and lq.full


def test_factorisation_detection():
    import paper_2603_01122_b200 as G
    from paper_2603_01122_b200.tables import _factorisation
    cs = G.ControlSet.grid(4, 24, 1.4)
    na, dv, heads, aidx = _factorisation(cs.v, cs.theta, np.arange(96))
    assert na == 4 and abs(dv - 1.4 / 3) < 1e-12 and len(heads) == 24
    assert sorted(aidx.ravel()) == list(range(96))
    keep = np.flatnonzero(cs.v <= 0.5)
    na, *_ = _factorisation(cs.v, cs.theta, keep)
    assert na == 2
    assert _factorisation(cs.v, cs.theta, np.arange(90)) is None


def test_window_geometry_bounds():
    """Every reachable cell after t steps lies in window t (host restatement of the
    kernel's window rule, checked on the oracle's exact positions)."""
    import torch
    import paper_2603_01122_b200 as G
    from paper_2603_01122_b200.tables import Geometry
    from oracle import predict as OP
    case = golden_io.PredictCase("ragged_w")
    W, H, res, org = case.grid
    spec = G.GridSpec(W, H, res, org)
    max_step = float(np.max(np.abs(np.stack([case.dispx, case.dispy]))))
    geo = Geometry(spec, case.steps, max_step, 0.0, torch.device("cpu"))
    out = OP.predict(case.z0, case.log_w, case.n, case.steps, case.dt, 0.0, case.seed, case.tables(),
                     case.beta_of, case.goal_xy_of, OP.Grid(W, H, res, org), prefix=case.prefix)
    z32 = (np.float32(case.z0[0]), np.float32(case.z0[1]))
    for t in range(case.steps):
        x0, y0, w, h = geo.window(z32, t)
        c = out["counts"][t]
        assert c.sum() == case.n
        assert c[y0:y0 + h, x0:x0 + w].sum() == case.n


def test_gcst_reads_reference_file_and_writes_identical_bytes(tmp_path):
    """gridio format row (f1): a file written by the reference loads, and a host-backed
    stack is written back byte-for-byte (header <4sIIII5d + row-major float64 layers)."""
    from paper_2603_01122_b200 import gridio
    src = os.path.join(golden_io.GOLDEN, "stack_ref.grd")
    st = gridio.load_stack(src)
    assert st.layers.shape == (3, 7, 12) and st.spec.origin == (-1.5, 2.0)
    assert st.dt == 0.2 and st.base_time == 4.5 and st.spec.resolution == 0.25
    out = tmp_path / "w.grd"
    gridio.save_stack(st, out)
    assert open(src, "rb").read() == open(out, "rb").read()
    with pytest.raises(ValueError):
        open(tmp_path / "bad.grd", "wb").write(b"XXXX" + b"\0" * 60)
        gridio.load_stack(tmp_path / "bad.grd")


def test_disc_offsets_order():
    import paper_2603_01122_b200 as G
    from paper_2603_01122_b200.occupancy import disc_offsets
    offs = disc_offsets(G.GridSpec(10, 10, 0.1), 0.25)
    assert offs[0].tolist() == [-1, -2] and len(offs) == 21
    assert (np.diff(offs[:, 1]) >= 0).all()
