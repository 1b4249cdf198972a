"""Fused region kernels vs the reference (golden) and the oracle at config sizes."""

import numpy as np
import pytest
import torch

import paper_2407_18352_b200 as sm
from goldens import arrays, infer_layers
from oracle import c_oracle, oracle
from paper_2407_18352_b200 import _native, workloads

pytestmark = pytest.mark.gpu


def model_of(layers, precision="fp32"):
    return sm.Model(layers[0][0].shape[1], layers[-1][0].shape[0],
                    [sm.DenseLayer(w, b, a) for w, b, a in layers], precision=precision)


def run_region(wl, tmp_path, **rt_kw):
    sm.save_model(wl.model, tmp_path / wl.spec.name)
    with sm.Runtime(**rt_kw) as rt:
        out = rt.invoke_region(rt.register_region(wl.descriptor(str(tmp_path / wl.spec.name))))
    return out


def test_options_region_golden(cuda, tmp_path):
    a = arrays()
    layers, _, _ = infer_layers("c1_options")
    recs = a["region_options_recs"]
    n = recs.shape[0]
    wl = workloads.make("options", n)
    wl.arrays["recs"] = recs
    wl.layers, wl.model = layers, model_of(layers)
    wl.to_device()
    assert _native.model_path(sm.models.device_model(wl.model, cuda)) == 1  # fused exact kernel
    run_region(wl, tmp_path)
    assert wl.buffers["price"].to_numpy().tobytes() == a["region_options_price"].tobytes()


def test_stencil_trajectory_golden(cuda, tmp_path):
    a = arrays()
    sm.save_model(sm.jacobi_model(0.25), tmp_path / "jm")
    f0 = a["region_stencil_field0"]
    t, tnew = sm.ArrayBuffer.from_numpy(f0), sm.ArrayBuffer.from_numpy(f0)
    env = {"N": 32, "M": 32}
    desc = sm.RegionDescriptor(
        name="stencil", accurate_fn=lambda: None,
        ml=sm.parse_directive(f'ml(infer) in(t) out(tnew) model("{tmp_path / "jm"}")'),
        in_maps=[sm.BoundMap(sm.parse_directive("functor(ifnctr: [i, j, 0:5] = (([i-1, j], [i+1, j], [i, j-1:j+2])))"),
                             sm.parse_directive("map(to: ifnctr(t[1:N-1, 1:M-1]))", env).targets[0], t)],
        out_maps=[sm.BoundMap(sm.parse_directive("functor(ofnctr: [i, j, 0:1] = ([i, j]))"),
                              sm.parse_directive("map(from: ofnctr(tnew[1:N-1, 1:M-1]))", env).targets[0], tnew)])
    with sm.Runtime() as rt:
        h = rt.register_region(desc)
        for _ in range(100):
            rt.invoke_region(h)
            t.view().copy_(tnew.view())
    assert t.to_numpy().tobytes() == a["region_stencil_final"].tobytes()


def test_weather_region_golden(cuda, tmp_path):
    a = arrays()
    layers, _, _ = infer_layers("c5_weather")
    wl = workloads.make("miniweather", 18 * 22)
    wl.arrays = {"state": a["region_weather_state"], "state_new": np.zeros((4, 20, 24), np.float32)}
    wl.env = {"NX": 20, "NZ": 24}
    wl.layers, wl.model = layers, model_of(layers)
    wl.to_device()
    run_region(wl, tmp_path)
    assert wl.buffers["state_new"].to_numpy().tobytes() == a["region_weather_new"].tobytes()


@pytest.mark.parametrize("flags", ["fused", "checked", "unfused"])
def test_options_full_size_bitwise(cuda, tmp_path, flags):
    wl = workloads.make("options")
    wl.to_device()
    if flags == "unfused":
        fi, fo, ti, to = wl.functors()
        rt = sm.Runtime()
        # drive the native call directly with FORCE_UNFUSED
        from paper_2407_18352_b200.bridge import _views_for, build_plan
        pin = build_plan([_views_for(fi, ti, wl.buffers["recs"])], "to")
        pout = build_plan([_views_for(fo, to, wl.buffers["price"])], "from")
        st = torch.zeros(1, dtype=torch.int32, device="cuda")
        h = sm.models.device_model(wl.model, cuda)
        _native.region_infer(pin.handle, *pin.ptrs_and_dtypes(), pout.handle, *pout.ptrs_and_dtypes(),
                             h, 0, pin.n_rows, _native.FORCE_UNFUSED, None,
                             torch.cuda.current_stream().cuda_stream, st.data_ptr())
        assert st.item() == 0
    else:
        run_region(wl, tmp_path, commit=flags)
    want, finite = c_oracle.mlp_f32(wl.layers, wl.arrays["recs"])
    assert finite
    assert wl.buffers["price"].to_numpy().tobytes() == want[:, 0].tobytes()


def test_weather_full_size_bitwise_bands(cuda, tmp_path):
    wl = workloads.make("miniweather")
    wl.to_device()
    run_region(wl, tmp_path)
    got = wl.buffers["state_new"].to_numpy()
    state = wl.arrays["state"]
    fi, fo, _, _ = wl.functors()
    for r0, r1 in ((1, 33), (2000, 2016), (4060, 4095)):
        band = sm.parse_directive(f"map(to: halo(state[{r0}:{r1}, 1:2047]))").targets[0]
        x = oracle.gather(fi, band, state.reshape(-1), state.shape, (4096 * 2048, 2048, 1)).reshape(-1, 36)
        y, finite = c_oracle.mlp_f32(wl.layers, x)
        assert finite
        want = y.reshape(r1 - r0, 2046, 4).transpose(2, 0, 1)
        assert got[:, r0:r1, 1:2047].tobytes() == np.ascontiguousarray(want).tobytes(), (r0, r1)
    # nothing outside the interior written
    assert not got[:, 0, :].any() and not got[:, -1, :].any() and not got[:, :, 0].any() and not got[:, :, -1].any()


def test_sharded_runtimes_cover_the_sweep(cuda, tmp_path):
    wl = workloads.make("options", 10_001)
    wl.to_device()
    sm.save_model(wl.model, tmp_path / "m")
    for rank in range(3):
        with sm.Runtime(shard=(rank, 3)) as rt:
            rt.invoke_region(rt.register_region(wl.descriptor(str(tmp_path / "m"))))
    want, _ = c_oracle.mlp_f32(wl.layers, wl.arrays["recs"])
    assert wl.buffers["price"].to_numpy().tobytes() == want[:, 0].tobytes()


@pytest.mark.parametrize("nz,commit,launches", [(132, "fused", 1), (132, "checked", 2), (130, "fused", 1),
                                                (66, "fused", 1)])
def test_weather_exact_kernels_bitwise(cuda, tmp_path, nz, commit, launches):
    """The TMA-ring exact stencil kernel (16-B multiple row pitch: 132, 66 is
    not -> the per-point fused kernel) and the per-point kernel (pitch 130)
    are both the oracle bit for bit, under both commits."""
    nx = 37
    wl = workloads.make("miniweather", (nx - 2) * (nz - 2))
    st = np.stack([workloads._bumps(nx, nz, k) for k in range(4)]).astype(np.float32)
    wl.arrays = {"state": st, "state_new": np.zeros_like(st)}
    wl.env = {"NX": nx, "NZ": nz}
    wl.to_device()
    n0 = _native.launch_count()
    run_region(wl, tmp_path, commit=commit)
    assert _native.launch_count() - n0 == launches
    fi, fo, ti, to = wl.functors()
    x = oracle.gather(fi, ti, st.reshape(-1), st.shape, (nx * nz, nz, 1)).reshape(-1, 36)
    y, _ = c_oracle.mlp_f32(wl.layers, x)
    want = np.zeros_like(st)
    want[:, 1:-1, 1:-1] = y.reshape(nx - 2, nz - 2, 4).transpose(2, 0, 1)
    assert wl.buffers["state_new"].to_numpy().reshape(st.shape).tobytes() == want.tobytes()
