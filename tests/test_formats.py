"""On-disk formats are byte-compatible with the reference writers (golden)."""

import json

import numpy as np

from goldens import arrays, infer_layers, meta
from paper_2407_18352_b200 import srdb
from paper_2407_18352_b200.models import DenseLayer, Model, load_model, save_model


def c1_model():
    layers, _, _ = infer_layers("c1_options")
    return Model(5, 1, [DenseLayer(w, b, a) for w, b, a in layers])


def test_model_files_byte_identical(tmp_path):
    save_model(c1_model(), tmp_path / "m")
    assert (tmp_path / "m" / "model.json").read_text() == meta()["model_json"]
    assert (tmp_path / "m" / "weights.bin").read_bytes() == arrays()["model_weights_bin"].tobytes()
    m = load_model(tmp_path / "m")
    for a, b in zip(m.layers, c1_model().layers):
        assert a.weights.tobytes() == b.weights.tobytes() and a.activation == b.activation


def test_bf16_hint_round_trip(tmp_path):
    m = c1_model()
    m.precision = "bf16"
    save_model(m, tmp_path / "m")
    assert json.loads((tmp_path / "m" / "model.json").read_text())["precision"] == "bf16"
    assert load_model(tmp_path / "m").precision == "bf16"


def test_srdb_bytes_identical(tmp_path):
    a = arrays()
    with srdb.open_db(tmp_path / "db", "create") as db:
        for k in range(3):
            assert db.append_record("stencil", a[f"srdb_x{k}"], a[f"srdb_y{k}"], 1000 + k) == k
    for which in ("inputs.bin", "outputs.bin", "times.bin"):
        got = (tmp_path / "db" / "regions" / "stencil" / which).read_bytes()
        assert got == a["srdb_" + which.replace(".", "_")].tobytes(), which
    man = json.loads((tmp_path / "db" / "manifest.json").read_text())
    man["regions"][0]["created_utc"] = "<nondeterministic>"
    assert man == meta()["srdb_manifest"]
    with srdb.open_db(tmp_path / "db", "read") as db:
        recs = db.read_records("stencil")
        assert [r.elapsed_ns for r in recs] == [1000, 1001, 1002]
        assert np.array_equal(recs[1].inputs.to_numpy(), a["srdb_x1"])


def test_cnn_model_v2_round_trip(tmp_path):
    from paper_2407_18352_b200 import workloads
    from paper_2407_18352_b200.models import Conv2dLayer, MaxPool2dLayer
    m = workloads.make("particlefilter", 2).model
    save_model(m, tmp_path / "pf")
    man = json.loads((tmp_path / "pf" / "model.json").read_text())
    assert man["version"] == 2 and man["input_shape"] == [1, 128, 128]
    assert [L.get("kind") for L in man["layers"]] == ["conv2d", "maxpool2d", "dense", "dense"]
    m2 = load_model(tmp_path / "pf")
    assert isinstance(m2.layers[0], Conv2dLayer) and isinstance(m2.layers[1], MaxPool2dLayer)
    assert m2.dims == [16384, 2048, 512, 128, 2]
    for a_, b_ in zip(m.layers, m2.layers):
        if hasattr(a_, "weights"):
            assert a_.weights.tobytes() == b_.weights.tobytes()


def test_srdb_read_by_reference_trainer(tmp_path):
    """The trainer's own reader (trainer/src/smlrt_train/srdb_reader.py:50-82)
    reads a database this runtime wrote (build container only: the reference
    checkout is not on the GPU boxes)."""
    import importlib.util
    import pytest
    path = "/root/reference/pkg/trainer/src/smlrt_train/srdb_reader.py"
    import os
    if not os.path.exists(path):
        pytest.skip("reference trainer not present")
    import sys
    import types
    pkg = types.ModuleType("smlrt_train")
    pkg.__path__ = [os.path.dirname(path)]
    sys.modules.setdefault("smlrt_train", pkg)
    spec = importlib.util.spec_from_file_location("smlrt_train.srdb_reader", path)
    reader = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(reader)
    rng = np.random.default_rng(0)
    xs = [rng.random((6, 6, 5), dtype=np.float32) for _ in range(4)]
    ys = [rng.random((6, 6, 1), dtype=np.float32) for _ in range(4)]
    with srdb.open_db(tmp_path / "db", "create") as db:
        for k in range(4):
            db.append_record("stencil", xs[k], ys[k], 10 + k)
    ins, outs, times = reader.read_region(tmp_path / "db", "stencil")
    assert ins.shape == (4, 6, 6, 5) and outs.shape == (4, 6, 6, 1)
    assert np.array_equal(ins, np.stack(xs)) and np.array_equal(outs, np.stack(ys))
    assert times.tolist() == [10, 11, 12, 13]
