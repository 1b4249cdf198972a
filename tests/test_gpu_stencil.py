"""Device-resident stencil driver (paper_2407_18352_b200.stencil): the
reference's acceptance criterion 3 (tests/test_acceptance.py:89-110, a
jacobi_model(0.25) surrogate tracks the accurate trajectory -- here exactly,
RMSE 0.0 at every step, as the survey measured for the reference) and its
interleave test (tests/test_bench.py:118-131: more accurate steps in the
schedule, less final error for an imperfect model)."""

import numpy as np
import pytest
import torch

import paper_2407_18352_b200 as sm
from paper_2407_18352_b200 import stencil, workloads

pytestmark = pytest.mark.gpu


def _field(n, m, seed, dev):
    return torch.from_numpy(workloads._bumps(n, m, seed)).to(dev)


def test_jacobi_surrogate_trajectory_exact(cuda, tmp_path):
    sm.save_model(sm.jacobi_model(0.25), tmp_path / "jm")
    run = stencil.run_stencil_device(_field(64, 48, 0, cuda), 100, str(tmp_path / "jm"), interleave=(0, 1))
    assert run.surrogate_calls == 100 and run.accurate_calls == 0
    assert max(run.per_step_rmse) == 0.0


def test_interleaving_reduces_final_error(cuda, tmp_path):
    # an imperfect ("drifty") surrogate: jacobi with the centre weight off by 2 %
    model = sm.jacobi_model(0.25)
    w = model.layers[0].weights.copy()
    w[0, 3] += np.float32(0.02)
    drifty = sm.Model(5, 1, [sm.DenseLayer(w, model.layers[0].bias, "identity")])
    sm.save_model(drifty, tmp_path / "drifty")
    finals = {}
    for sched in [(0, 1), (1, 1), (3, 1)]:
        errs = [stencil.run_stencil_device(_field(16, 16, seed, cuda), 40, str(tmp_path / "drifty"),
                                           interleave=sched).per_step_rmse[-1] for seed in range(5)]
        finals[sched] = float(np.mean(errs))
    assert finals[(3, 1)] <= finals[(1, 1)] <= finals[(0, 1)]
    assert finals[(1, 1)] < finals[(0, 1)]


def test_schedule_call_counts(cuda, tmp_path):
    sm.save_model(sm.jacobi_model(0.25), tmp_path / "jm")
    run = stencil.run_stencil_device(_field(16, 16, 1, cuda), 12, str(tmp_path / "jm"), interleave=(1, 2))
    assert run.accurate_calls == 4 and run.surrogate_calls == 8
    assert max(run.per_step_rmse) == 0.0
