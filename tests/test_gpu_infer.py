"""Forward pass on the GPU vs the reference's infer (golden) and the oracle."""

import numpy as np
import pytest
import torch

import paper_2407_18352_b200 as sm
from goldens import infer_layers, meta
from paper_2407_18352_b200.errors import NonFiniteOutputError, ShapeMismatchError

pytestmark = pytest.mark.gpu


def model_of(layers):
    return sm.Model(layers[0][0].shape[1], layers[-1][0].shape[0],
                    [sm.DenseLayer(w, b, a) for w, b, a in layers])


@pytest.mark.parametrize("name", [m["name"] for m in meta()["infer"]])
def test_infer_goldens(cuda, name):
    layers, x, y = infer_layers(name)
    got = sm.infer(model_of(layers), x)
    if any(a == "tanh" for _, _, a in layers):
        assert np.max(np.abs(got - y)) <= 1e-5 * max(1.0, np.abs(y).max())
    else:
        assert got.tobytes() == y.tobytes(), np.abs(got - y).max()


def test_batch_independence_exact(cuda):
    rng = np.random.default_rng(11)
    layers = [(rng.normal(scale=0.5, size=(o, i)).astype(np.float32),
               rng.normal(scale=0.1, size=o).astype(np.float32), a)
              for i, o, a in ((5, 12, "relu"), (12, 12, "relu"), (12, 2, "identity"))]
    m = model_of(layers)
    x = rng.normal(size=(33, 5)).astype(np.float32)
    whole = sm.infer(m, x)
    rows = np.concatenate([sm.infer(m, x[k:k + 1]) for k in range(33)])
    assert np.array_equal(whole, rows)


def test_f64_round_trip_and_tensor_kinds(cuda):
    m = sm.Model(4, 4, [sm.DenseLayer(np.eye(4, dtype=np.float32), np.zeros(4, np.float32), "identity")])
    x = np.random.default_rng(0).normal(size=(6, 4))
    out = sm.infer(m, x)
    assert out.dtype == np.float64 and np.array_equal(out, x.astype(np.float32).astype(np.float64))
    t = sm.infer(m, sm.Tensor(torch.ones(2, 4, device="cuda")))
    assert isinstance(t, sm.Tensor) and t.data.is_cuda
    with pytest.raises(ShapeMismatchError):
        sm.infer(m, np.zeros((3, 5), np.float32))


def test_overflow_raises(cuda):
    m = sm.Model(1, 1, [sm.DenseLayer(np.array([[2.0]], np.float32), np.zeros(1, np.float32), "identity")])
    with pytest.raises(NonFiniteOutputError):
        sm.infer(m, np.full((1, 1), 3e38, np.float32))
    nan_relu = sm.Model(1, 1, [sm.DenseLayer(np.array([[1.0]], np.float32), np.zeros(1, np.float32), "relu")])
    with pytest.raises(NonFiniteOutputError):  # relu keeps NaN (np.maximum semantics)
        sm.infer(nan_relu, np.full((1, 1), np.nan, np.float32))
