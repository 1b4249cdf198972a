"""C4 ParticleFilter CNN: fused window-gather conv/pool front + exact dense
tail vs the reference-composed golden and the oracle (bitwise)."""

import numpy as np
import pytest
import torch

import paper_2407_18352_b200 as sm
from goldens import arrays
from oracle import oracle
from paper_2407_18352_b200 import _native, workloads
from paper_2407_18352_b200.models import Conv2dLayer, DenseLayer, MaxPool2dLayer, Model

pytestmark = pytest.mark.gpu


def golden_model():
    a = arrays()
    return Model(16384, 2, [Conv2dLayer(a["cnn_conv_w"], a["cnn_conv_b"], 8, 8, "relu"), MaxPool2dLayer(2),
                            DenseLayer(a["cnn_fc_W0"], a["cnn_fc_b0"], "relu"),
                            DenseLayer(a["cnn_fc_W1"], a["cnn_fc_b1"], "identity")], input_shape=(1, 128, 128))


def run(wl, tmp_path, model=None, **kw):
    sm.save_model(model or wl.model, tmp_path / "pf")
    with sm.Runtime(**kw) as rt:
        rt.invoke_region(rt.register_region(wl.descriptor(str(tmp_path / "pf"))))
    return wl.buffers["locs"].to_numpy()


def test_cnn_region_golden(cuda, tmp_path):
    a = arrays()
    wl = workloads.make("particlefilter", 3)
    wl.arrays["frames"] = a["cnn_frames"]
    wl.to_device()
    m = golden_model()
    assert _native.model_path(sm.models.device_model(m, cuda)) == 4
    got = run(wl, tmp_path, m)
    assert got.tobytes() == a["cnn_y"].tobytes()


def test_cnn_infer_dense_batch(cuda):
    a = arrays()
    x = a["cnn_frames"][:, 16:144, 16:144].reshape(3, -1)
    y = sm.infer(golden_model(), x)
    assert y.tobytes() == a["cnn_y"].tobytes()


@pytest.mark.parametrize("commit", ["fused", "checked"])
def test_cnn_region_matches_oracle(cuda, tmp_path, commit):
    wl = workloads.make("particlefilter", 700)
    wl.to_device()
    got = run(wl, tmp_path, commit=commit)
    x = wl.arrays["frames"][:, 16:144, 16:144].reshape(700, -1)
    want, finite = oracle.cnn_forward(workloads.cnn_layers(), x, (1, 128, 128))
    assert finite and got.tobytes() == want.tobytes()


def test_cnn_full_size_subsample(cuda, tmp_path):
    wl = workloads.make("particlefilter")
    wl.to_device()
    got = run(wl, tmp_path)
    idx = np.arange(0, wl.elements, 61)
    x = wl.arrays["frames"][idx, 16:144, 16:144].reshape(len(idx), -1)
    want, _ = oracle.cnn_forward(workloads.cnn_layers(), x, (1, 128, 128))
    assert got[idx].tobytes() == want.tobytes()


def test_cnn_overlapped_chunks_bitwise(cuda):
    """The opt-in two-stream chunked CNN region (SMLRT_CNN_CHUNKS=3: conv
    front on a side stream, dense tail on the caller's) is bitwise the oracle,
    including a ragged last chunk (run in a subprocess: the switch is read once)."""
    import os
    import subprocess
    import sys
    code = ("import sys, pathlib, tempfile, numpy as np; sys.path.insert(0, '.'); sys.path.insert(0, 'tests');"
            "import paper_2407_18352_b200 as sm; from paper_2407_18352_b200 import workloads; from oracle import oracle;"
            "n = 3 * 4096 + 123; wl = workloads.make('particlefilter', n); wl.to_device();"
            "d = pathlib.Path(tempfile.mkdtemp()); sm.save_model(wl.model, d / 'pf');"
            "rt = sm.Runtime(); rt.invoke_region(rt.register_region(wl.descriptor(str(d / 'pf'))));"
            "got = wl.buffers['locs'].to_numpy(); idx = np.r_[0:50, 4090:4100, 8190:8200, n - 130:n];"
            "x = wl.arrays['frames'][idx, 16:144, 16:144].reshape(len(idx), -1);"
            "want, _ = oracle.cnn_forward(workloads.cnn_layers(), x, (1, 128, 128));"
            "assert got[idx].tobytes() == want.tobytes(); print('ok')")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env={**os.environ, "SMLRT_CNN_CHUNKS": "3"},
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]
