"""bf16 halo-stencil regions on tcgen05 (stencil_tc.cu): the MiniWeather
region at precision "bf16" -- layer 1 on tf32 and layer 2 on bf16 warp-level
MMAs fed from a TMA ring -- against the fp32 oracle (SURVEY.md 8(d) bf16 tolerance: max-abs
<= 2e-2 max|ref|, RMSE/RMS <= 1e-2) and against an emulation of its
quantisation points (max-abs <= 2e-3 max|ref|)."""

import numpy as np
import pytest
import torch

import paper_2407_18352_b200 as sm
from oracle import c_oracle
from paper_2407_18352_b200 import _native, workloads
from paper_2407_18352_b200.errors import NonFiniteOutputError

pytestmark = pytest.mark.gpu


def _bf16(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(torch.bfloat16).to(torch.float64).numpy()


def _halo_features(state):
    """[NX-2, NZ-2, 36] features of the MiniWeather functor (v, di, dj order)."""
    V, NX, NZ = state.shape
    cols = [state[v, 1 + di - 1:NX - 1 + di - 1, 1 + dj - 1:NZ - 1 + dj - 1]
            for v in range(V) for di in range(3) for dj in range(3)]
    return np.stack(cols, -1).reshape(-1, 36)


def _tf32_trunc(a):
    u = np.ascontiguousarray(a, np.float32).view(np.uint32) & np.uint32(0xFFFFE000)
    return u.view(np.float32).astype(np.float64)


def _tf32_rne(a):
    u = np.ascontiguousarray(a, np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0xFFF + ((u >> 13) & 1)) & 0xFFFFE000
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def _emulate(layers, x):
    """the kernel's quantisation points: tf32 features (the MMA keeps their top
    19 bits) and W1 (rounded), f32 accumulation from the bias, activation,
    bf16 hidden and W2, f32 accumulation"""
    (w1, b1, a1), (w2, b2, a2) = layers
    h = _tf32_trunc(x) @ _tf32_rne(w1).T + b1
    h = np.maximum(h, 0) if a1 == "relu" else (np.tanh(h) if a1 == "tanh" else h)
    y = _bf16(h) @ _bf16(w2).T + b2
    return np.maximum(y, 0) if a2 == "relu" else (np.tanh(y) if a2 == "tanh" else y)


def _run(wl, tmp_path, **kw):
    wl.to_device()
    sm.save_model(wl.model, tmp_path / "mw")
    with sm.Runtime(**kw) as rt:
        rt.invoke_region(rt.register_region(wl.descriptor(str(tmp_path / "mw"))))
    return wl.buffers["state_new"].to_numpy()


def _check(wl, got, emulate=True):
    state = wl.arrays["state"]
    x = _halo_features(state)
    y = np.stack([got[v, 1:-1, 1:-1].reshape(-1) for v in range(4)], -1).astype(np.float64)
    ref, _ = c_oracle.mlp_f32(wl.layers, x)
    ref = ref.astype(np.float64)
    err = np.abs(y - ref)
    scale = np.abs(ref).max()
    assert err.max() <= 2e-2 * scale, (err.max(), scale)
    assert np.sqrt(np.mean(err ** 2)) / np.sqrt(np.mean(ref ** 2)) <= 1e-2
    if not emulate:
        return
    # vs the emulated quantisation: equal up to f32 summation order, which can
    # flip a hidden unit's bf16 rounding (one bf16 ulp of h times a W2 weight)
    emu = _emulate(wl.layers, x)
    d = np.abs(y - emu)
    assert np.sqrt(np.mean(d ** 2)) <= 1e-4 * np.sqrt(np.mean(emu ** 2))
    assert d.max() <= 1.5e-2 * np.abs(emu).max()
    # the border (not in the sweep) is untouched
    assert (got[:, 0, :] == 0).all() and (got[:, -1, :] == 0).all()
    assert (got[:, :, 0] == 0).all() and (got[:, :, -1] == 0).all()


@pytest.mark.parametrize("nx,nz", [(40, 132), (67, 252), (6, 8)])
@pytest.mark.parametrize("commit", ["fused", "checked"])
def test_stencil_tc_matches_oracle(cuda, tmp_path, nx, nz, commit):
    """ragged column blocks (126 per CTA) and row blocks, few-column grids (the row
    pitch must be a multiple of 4 elements: the TMA ring's 16-B stride rule)"""
    wl = workloads.make("miniweather_bf16", (nx - 2) * (nz - 2))
    st = np.stack([workloads._bumps(nx, nz, k) + np.random.default_rng(k).normal(0, 0.05, (nx, nz))
                   .astype(np.float32) for k in range(4)]).astype(np.float32)
    wl.arrays = {"state": st, "state_new": np.zeros_like(st)}
    wl.env = {"NX": nx, "NZ": nz}
    n0 = _native.launch_count()
    got = _run(wl, tmp_path, commit=commit)
    # one stencil kernel (+ the gated scatter of the checked commit), not the 4-launch layer chain
    assert _native.launch_count() - n0 == (1 if commit == "fused" else 2)
    _check(wl, got)


def test_stencil_tc_full_size(cuda, tmp_path):
    wl = workloads.make("miniweather_bf16")
    got = _run(wl, tmp_path)
    _check(wl, got)


def _mw(nx, nz):
    wl = workloads.make("miniweather_bf16", (nx - 2) * (nz - 2))
    st = np.stack([workloads._bumps(nx, nz, k) for k in range(4)]).astype(np.float32)
    wl.arrays = {"state": st, "state_new": np.zeros_like(st)}
    wl.env = {"NX": nx, "NZ": nz}
    return wl


@pytest.mark.parametrize("nz,launches", [(132, 2), (130, 3)])  # stencil kernel / layer chain (last layer fused), + the gated scatter
@pytest.mark.parametrize("bad", [np.inf, np.nan])
def test_stencil_nonfinite(cuda, tmp_path, nz, launches, bad):
    wl = _mw(40, nz)
    wl.arrays["state"][2, 10, 20] = bad
    wl.to_device()
    sm.save_model(wl.model, tmp_path / "mw")
    n0 = _native.launch_count()
    with sm.Runtime(commit="checked") as rt:
        with pytest.raises(NonFiniteOutputError):
            rt.invoke_region(rt.register_region(wl.descriptor(str(tmp_path / "mw"))))
    assert _native.launch_count() - n0 == launches
    assert (wl.buffers["state_new"].to_numpy() == 0).all()


def test_stencil_unaligned_pitch_uses_chain(cuda, tmp_path):
    """A row pitch that is not a multiple of 4 elements cannot be a TMA
    stride: the region runs on the generic layer chain, same tolerance."""
    wl = _mw(20, 130)
    n0 = _native.launch_count()
    got = _run(wl, tmp_path)
    assert _native.launch_count() - n0 == 3  # gather, one GEMM (36->8 with the 8->4 layer in its epilogue), scatter
    _check(wl, got, emulate=False)  # the chain quantises to bf16 throughout


def test_stencil_f64_takes_the_chain(cuda, tmp_path):
    wl = _mw(20, 132)
    wl.arrays = {k: v.astype(np.float64) for k, v in wl.arrays.items()}
    n0 = _native.launch_count()
    got = _run(wl, tmp_path)
    assert _native.launch_count() - n0 == 3 and got.dtype == np.float64
    _check(wl, got.astype(np.float32), emulate=False)
