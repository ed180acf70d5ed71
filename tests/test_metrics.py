"""dataset.mape mirror (host) against the reference's golden MAPE, its error
behaviour (dataset.py:229-248), and the device-side evaluate() path."""

import numpy as np
import pytest

from conftest import unpack_records
from paper_2303_11733_b200 import metrics
from paper_2303_11733_b200.errors import LengthMismatch, ZeroActual
from paper_2303_11733_b200.types import TargetVector


def test_mape_matches_reference_golden(golden, golden_next):
    from test_oracle_golden import _norm, mlp_params
    from oracle import dippm_oracle as O
    recs = unpack_records(golden)
    params = mlp_params(golden_next, "mlp32")
    preds = [TargetVector(*O.mlp_predict(params, _norm(golden), r[3])) for r in recs]
    m = metrics.mape(preds, [TargetVector(*r[4]) for r in recs])
    assert np.allclose([m.latency, m.memory, m.energy, m.overall], golden_next["mape_mlp32"], rtol=1e-12)


def test_mape_errors():
    t = TargetVector(1.0, 2.0, 3.0)
    with pytest.raises(LengthMismatch):
        metrics.mape([t], [])
    with pytest.raises(LengthMismatch):
        metrics.mape([], [])
    with pytest.raises(ZeroActual):
        metrics.mape([t], [TargetVector(1.0, 0.0, 3.0)])
    assert metrics.mape([t], [t]).overall == 0.0


@pytest.mark.gpu
@pytest.mark.parametrize("arch", ["sage", "mlp"])
def test_device_evaluate_equals_host_mape(golden, golden_next, arch):
    from paper_2303_11733_b200 import gnn
    from test_gpu_model import _model, _records
    from test_gpu_mlp import _mlp
    model = _model(golden, "h32") if arch == "sage" else _mlp(golden, golden_next, "mlp32")
    recs = _records(golden)
    host = metrics.mape(gnn.predict_records(model, recs), [r.target for r in recs])
    dev, loss = metrics.evaluate(model, recs, batch_size=7, with_loss=True)  # several batches
    for a, b in zip(dev.as_dict().values(), host.as_dict().values()):
        assert abs(a - b) <= 1e-6 * max(1.0, abs(b))
    assert abs(loss - gnn.batch_loss(model, recs)) <= 1e-6
    rep = metrics.eval_report(model, recs)
    assert rep["n"] == len(recs) and set(rep["mape"]) == {"latency", "memory", "energy", "overall"}
