"""First-call overhead estimator (reference tenhost/overhead.py:76-175)."""

import csv

import pytest

from paper_2510_01495_b200 import overhead
from paper_2510_01495_b200.errors import ConfigError, EstimationError


def test_argument_validation():
    with pytest.raises(ConfigError):
        overhead.estimate_overhead("native-loop", 10)
    with pytest.raises(ConfigError):
        overhead.estimate_overhead(size=10, experiment="mttkrp")
    with pytest.raises(ConfigError):
        overhead.estimate_overhead(size=10, repeats=0)


def test_csv_format(tmp_path):
    est = overhead.OverheadEstimate("b200", "n=10", 0.5, 0.25, 0.25, 3)
    p = tmp_path / "o.csv"
    overhead.write_overhead_csv([est], p)
    rows = list(csv.reader(open(p)))
    assert rows[0] == list(overhead.OVERHEAD_COLUMNS)
    assert rows[1] == ["b200", "n=10", "0.5", "0.25", "0.25", "3"]


def test_failed_repeats_are_discarded_and_reported():
    """Without a GPU every child fails (the library raises DeviceError): each repeat is reported
    and discarded, and the estimate raises EstimationError, as in the reference."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible: the children succeed (covered by the gpu test)")
    msgs = []
    with pytest.raises(EstimationError):
        overhead.estimate_overhead(size=1000, n_trials=2, repeats=2, report=msgs.append, timeout_s=120)
    assert len(msgs) == 2 and all("discarded" in m for m in msgs)


@pytest.mark.gpu
def test_first_call_overhead_on_gpu():
    for exp, size in (("dot", 100000), ("ttv", 100)):
        est = overhead.estimate_overhead(size=size, experiment=exp, n_trials=5, repeats=2, timeout_s=300)
        assert est.repeats == 2
        assert est.first_call_mean_s > est.steady_mean_s > 0
        assert est.overhead_s == pytest.approx(est.first_call_mean_s - est.steady_mean_s)
