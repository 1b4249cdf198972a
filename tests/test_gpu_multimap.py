"""Multi-map regions on the GPU (runtime.py:312-357): several in-maps over
different arrays (f32 and f64) concatenated on F in in_maps + inout_maps
order, outputs split over out_maps + inout_maps in that order, an inout map
read before it is written (snapshot semantics).  Every kernel family is
checked against the oracle's `region` (the reference's _run_surrogate
restated): fp32-exact paths bitwise, bf16 within the survey tolerance."""

import numpy as np
import pytest

import paper_2407_18352_b200 as sm
from oracle import oracle
from paper_2407_18352_b200 import _native, workloads

pytestmark = pytest.mark.gpu


def strides(a):
    return tuple(int(np.prod(a.shape[k + 1:])) for k in range(a.ndim))


def run_both(tmp_path, model, layers, arrays, ins, outs, inouts, env, precision=None):
    """arrays: name -> numpy array; ins/outs/inouts: [(functor text, map target text)].
    Runs the GPU region and the oracle region; returns (gpu arrays, oracle arrays)."""
    bufs = {k: sm.ArrayBuffer.from_numpy(v) for k, v in arrays.items()}

    def bind(specs, kind):
        out = []
        for ftxt, ttxt in specs:
            f = sm.parse_directive(ftxt)
            t = sm.parse_directive(f"map({kind}: {ttxt})", env).targets[0]
            out.append((f, t))
        return out

    bi, bo, bio = bind(ins, "to"), bind(outs, "from"), bind(inouts, "to")
    names = lambda b: ", ".join(t.array for _, t in b)  # noqa: E731
    clause = "ml(infer)"
    if bi:
        clause += f" in({names(bi)})"
    if bo:
        clause += f" out({names(bo)})"
    if bio:
        clause += f" inout({names(bio)})"
    mdir = tmp_path / "m"
    sm.save_model(model, mdir)
    desc = sm.RegionDescriptor(
        name="mm", accurate_fn=lambda: None, ml=sm.parse_ml_clause(clause + f' model("{mdir}")'),
        in_maps=[sm.BoundMap(f, t, bufs[t.array]) for f, t in bi],
        out_maps=[sm.BoundMap(f, t, bufs[t.array]) for f, t in bo],
        inout_maps=[sm.BoundMap(f, t, bufs[t.array]) for f, t in bio], env=env)
    with sm.Runtime(precision=precision) as rt:
        rt.invoke_region(rt.register_region(desc))
    got = {k: b.to_numpy() for k, b in bufs.items()}
    want = {k: v.copy() for k, v in arrays.items()}
    m = lambda b: [(f, t, want[t.array].reshape(-1), want[t.array].shape, strides(want[t.array]))  # noqa: E731
                   for f, t in b]
    if model.layers and isinstance(model.layers[0], sm.models.Conv2dLayer):
        # CNN: oracle gather -> cnn_forward -> scatter per out map
        xs = [oracle.gather(f, t, d, sh, st).reshape(-1, f.feature_count) for f, t, d, sh, st in m(bi + bio)]
        x = np.concatenate(xs, axis=1) if len(xs) > 1 else xs[0]
        y, _ = oracle.cnn_forward(layers, x, model.input_shape)
        col = 0
        for f, t, d, sh, st in m(bo + bio):
            oracle.scatter(f, t, y[:, col:col + f.feature_count], d, sh, st)
            col += f.feature_count
    else:
        oracle.region(m(bi + bio), m(bo + bio), layers)
    return got, want


def dense_model(dims, precision="fp32", act="relu"):
    layers = workloads.init_weights(dims, act)
    return sm.Model(dims[0], dims[-1], [sm.DenseLayer(w, b, a) for w, b, a in layers], precision=precision), layers


def halo_fields(nx, nz, seed):
    rng = np.random.default_rng(seed)
    return rng.uniform(-1, 1, size=(2, nx, nz))


def test_exact_fused_two_in_two_out_mixed_dtypes(cuda, tmp_path):
    """36-8-4 (the fused C5 instantiation): 18 halo features from an f32
    array + 18 from an f64 array; G = 4 split 2 + 2 over an f32 and an f64
    output array."""
    nx, nz = 37, 70
    env = {"NX": nx, "NZ": nz}
    arrays = {"p": halo_fields(nx, nz, 1).astype(np.float32), "q": halo_fields(nx, nz, 2),
              "o1": np.full((2, nx, nz), 7.0, np.float32), "o2": np.full((2, nx, nz), -3.0)}
    model, layers = dense_model([36, 8, 4])
    h = "[i, j, 0:2, 0:3, 0:3] = ([0:2, i-1:i+2, j-1:j+2])"
    got, want = run_both(
        tmp_path, model, layers, arrays,
        ins=[(f"functor(hp: {h})", "hp(p[1:NX-1, 1:NZ-1])"), (f"functor(hq: {h})", "hq(q[1:NX-1, 1:NZ-1])")],
        outs=[("functor(o1f: [i, j, 0:2] = ([0, i, j], [1, i, j]))", "o1f(o1[1:NX-1, 1:NZ-1])"),
              ("functor(o2f: [i, j, 0:2] = ([0, i, j], [1, i, j]))", "o2f(o2[1:NX-1, 1:NZ-1])")],
        inouts=[], env=env)
    assert sm.models.device_model(model, cuda) is not None
    for k in ("o1", "o2"):
        assert np.array_equal(got[k], want[k]), k
    assert (got["o1"][:, 0, :] == 7.0).all() and (got["o2"][:, :, -1] == -3.0).all()  # off-sweep untouched


def test_exact_inout_map_reads_before_write(cuda, tmp_path):
    """5-64-32-1 (the fused C1 instantiation): 4 features from an f32 record
    array + 1 from an inout f64 column that also receives the output."""
    n = 5003
    rng = np.random.default_rng(3)
    arrays = {"recs": rng.uniform(0, 1, (n, 4)).astype(np.float32), "x": rng.uniform(0, 1, (n, 3))}
    model, layers = dense_model([5, 64, 32, 1])
    got, want = run_both(
        tmp_path, model, layers, arrays,
        ins=[("functor(r4: [k, 0:4] = ([k, 0:4]))", "r4(recs[0:N])")], outs=[],
        inouts=[("functor(xc: [k, 0:1] = ([k, 1]))", "xc(x[0:N])")], env={"N": n})
    assert np.array_equal(got["x"], want["x"])
    assert np.array_equal(got["x"][:, [0, 2]], arrays["x"][:, [0, 2]])
    assert not np.array_equal(got["x"][:, 1], arrays["x"][:, 1])


def test_exact_unfused_shape_two_in_maps(cuda, tmp_path):
    """A shape without a fused instantiation (7-48-24-3) through two in-maps
    and two out-maps."""
    n = 3001
    rng = np.random.default_rng(4)
    arrays = {"a": rng.uniform(-1, 1, (n, 5)).astype(np.float32), "b": rng.uniform(-1, 1, (2, n)),
              "y": np.zeros((n, 2), np.float32), "z": np.zeros(n)}
    model, layers = dense_model([7, 48, 24, 3])
    got, want = run_both(
        tmp_path, model, layers, arrays,
        ins=[("functor(fa: [k, 0:5] = ([k, 0:5]))", "fa(a[0:N])"), ("functor(fb: [k, 0:2] = ([0:2, k]))", "fb(b[0:N])")],
        outs=[("functor(fy: [k, 0:2] = ([k, 0], [k, 1]))", "fy(y[0:N])"), ("functor(fz: [k, 0:1] = ([k]))", "fz(z[0:N])")],
        inouts=[], env={"N": n})
    assert np.array_equal(got["y"], want["y"]) and np.array_equal(got["z"], want["z"])


def check_tol(got, ref):
    err = np.abs(got - ref)
    scale = np.abs(ref).max()
    rmse = np.sqrt(np.mean((got - ref) ** 2)) / np.sqrt(np.mean(ref ** 2))
    assert err.max() <= 2e-2 * scale, (err.max(), scale)
    assert rmse <= 1e-2, rmse


def test_tcgen05_two_in_maps_f32_f64(cuda, tmp_path):
    """Bonds model (16-256-128-1, bf16 tcgen05): 10 features from an f32
    array and 6 from an f64 array; the output into an f64 array."""
    n = 40_000
    rng = np.random.default_rng(5)
    arrays = {"a": rng.random((n, 10), dtype=np.float32), "b": rng.random((n, 6)), "v": np.zeros(n)}
    model, layers = dense_model([16, 256, 128, 1], "bf16")
    got, want = run_both(
        tmp_path, model, layers, arrays,
        ins=[("functor(fa: [k, 0:10] = ([k, 0:10]))", "fa(a[0:N])"), ("functor(fb: [k, 0:6] = ([k, 0:6]))", "fb(b[0:N])")],
        outs=[("functor(fv: [k, 0:1] = ([k]))", "fv(v[0:N])")], inouts=[], env={"N": n})
    check_tol(got["v"], want["v"])


def test_cnn_two_out_maps(cuda, tmp_path):
    """ParticleFilter CNN: the window functor in, the two outputs split over
    an f32 and an f64 array."""
    n = 37
    rng = np.random.default_rng(6)
    wl = workloads.make("particlefilter", n)
    arrays = {"frames": wl.arrays["frames"], "lx": np.zeros(n, np.float32), "ly": np.zeros(n)}
    got, want = run_both(
        tmp_path, wl.model, wl.layers, arrays,
        ins=[("functor(win: [k, 0:128, 0:128] = ([k, 16:144, 16:144]))", "win(frames[0:N])")],
        outs=[("functor(fx: [k, 0:1] = ([k]))", "fx(lx[0:N])"), ("functor(fy: [k, 0:1] = ([k]))", "fy(ly[0:N])")],
        inouts=[], env={"N": n})
    del rng
    assert np.array_equal(got["lx"], want["lx"]) and np.array_equal(got["ly"], want["ly"])
