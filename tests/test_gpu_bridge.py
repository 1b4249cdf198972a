"""GPU gather/scatter kernels vs the reference's golden vectors (bitwise)."""

import numpy as np
import pytest
import torch

import paper_2407_18352_b200 as sm
from goldens import arrays, case, functor, meta, target
from paper_2407_18352_b200 import errors

pytestmark = pytest.mark.gpu


def dev_array(data, shape, strides):
    return sm.ArrayBuffer(torch.from_numpy(np.ascontiguousarray(data)).cuda(), shape, strides)


def test_c1_corpus_bitwise(cuda):
    a = arrays()
    for i in range(len(meta()["c1"])):
        f, t, c = case("c1", i)
        got = sm.concretize_to(f, t, dev_array(a[f"c1_{i}_data"], c["shape"], c["strides"]))
        want = a[f"c1_{i}_out"]
        assert got.shape == want.shape and got.dtype == c["dtype"]
        assert got.to_numpy().tobytes() == want.tobytes(), i


def test_scatter_corpus_bitwise(cuda):
    a = arrays()
    for i in range(len(meta()["scatter"])):
        f, t, c = case("scatter", i)
        after = a[f"sc_{i}_after"]
        dst = dev_array(np.full(after.shape, -7.0, after.dtype), c["shape"], c["strides"])
        sm.scatter_from(f, t, sm.Tensor(torch.from_numpy(a[f"sc_{i}_payload"]).cuda()), dst)
        assert dst.data.cpu().numpy().tobytes() == after.tobytes(), i


def test_worked_example_and_interior_scatter(cuda):
    grid = sm.ArrayBuffer.from_numpy(np.arange(16, dtype=np.float32).reshape(4, 4))
    f = sm.parse_directive("functor(ifnctr: [i, j, 0:5] = ([i-1, j], [i+1, j], [i, j-1:j+2]))")
    t = sm.parse_directive("map(to: ifnctr(t[1:N-1, 1:M-1]))", {"N": 4, "M": 4}).targets[0]
    x = sm.concretize_to(f, t, grid)
    assert x.shape == (2, 2, 5)
    assert x.data[0, 0].tolist() == [1, 9, 4, 5, 6] and x.data[1, 1].tolist() == [6, 14, 9, 10, 11]
    dst = sm.ArrayBuffer.from_numpy(np.full((4, 4), -1.0, np.float32))
    g = sm.parse_directive("functor(ofnctr: [i, j, 0:1] = ([i, j]))")
    sm.scatter_from(g, t, sm.Tensor(torch.arange(4.0).reshape(2, 2, 1).cuda()), dst)
    after = dst.to_numpy()
    assert np.array_equal(after[1:3, 1:3], np.arange(4.0).reshape(2, 2))
    border = after.copy()
    border[1:3, 1:3] = -1
    assert (border == -1).all()


def test_golden_error_classes(cuda):
    for c in meta()["errors"]:
        f, t = functor(c["functor"]), target(c["target"])
        arr = sm.ArrayBuffer.from_numpy(np.arange(int(np.prod(c["shape"])), dtype=np.float32)
                                        .reshape(c["shape"]))

        def run():
            if c["op"] == "concretize":
                sm.concretize_to(f, t, arr)
            else:
                payload = torch.ones(tuple(s.count for s in t.slices) + f.feature_sizes).cuda()
                sm.scatter_from(f, t, sm.Tensor(payload), arr)

        if c["error"] is None:
            run()
        else:
            with pytest.raises(getattr(errors, c["error"])):
                run()


def test_column_major_and_f64_and_round_trip(cuda):
    base = np.asfortranarray(np.arange(16, dtype=np.float64).reshape(4, 4))
    arr = sm.ArrayBuffer(torch.from_numpy(base.ravel(order="K").copy()).cuda(), (4, 4), (1, 4))
    f = sm.parse_functor_decl("f: [i, j, 0:1] = ([i, j])")
    t = sm.parse_tensor_map("map(to: f(t[0:4, 0:4]))").targets[0]
    got = sm.concretize_to(f, t, arr)
    assert got.dtype == "f64" and np.array_equal(got.to_numpy()[..., 0], base)
    src = sm.ArrayBuffer.from_numpy(np.random.default_rng(3).normal(size=(6, 5)))
    t = sm.parse_tensor_map("map(to: f(a[1:5, 2:4]))").targets[0]
    x = sm.concretize_to(f, t, src)
    dst = sm.ArrayBuffer.zeros((6, 5), "f64")
    sm.scatter_from(f, t, x, dst)
    assert np.array_equal(dst.to_numpy()[1:5, 2:4], src.to_numpy()[1:5, 2:4])
    outside = dst.to_numpy().copy()
    outside[1:5, 2:4] = 0
    assert not outside.any()


def test_scatter_casts_f32_tensor_into_f64_array(cuda):
    f = sm.parse_functor_decl("f: [k, 0:1] = ([k])")
    t = sm.parse_tensor_map("map(from: f(a[0:8:2]))").targets[0]
    dst = sm.ArrayBuffer.zeros((8,), "f64")
    vals = torch.tensor([1.1, 2.2, 3.3, 4.4], dtype=torch.float32).reshape(4, 1).cuda()
    sm.scatter_from(f, t, sm.Tensor(vals), dst)
    want = np.zeros(8)
    want[0::2] = vals.cpu().numpy()[:, 0].astype(np.float64)
    assert np.array_equal(dst.to_numpy(), want)


def test_large_gather_matches_oracle(cuda):
    from oracle import oracle
    rng = np.random.default_rng(1)
    state = rng.normal(size=(4, 256, 300)).astype(np.float32)
    f = sm.parse_directive("functor(halo: [i, j, 0:4, 0:3, 0:3] = ([0:4, i-1:i+2, j-1:j+2]))")
    t = sm.parse_directive("map(to: halo(state[1:255, 1:299]))").targets[0]
    got = sm.concretize_to(f, t, sm.ArrayBuffer.from_numpy(state)).to_numpy()
    want = oracle.gather(f, t, state.reshape(-1), state.shape, (256 * 300, 300, 1))
    assert got.tobytes() == want.tobytes()
