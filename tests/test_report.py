"""CPU: the run report (src/io.cpp:156-253)."""
import pytest

from paper_1411_0814_b200 import rsm
from paper_1411_0814_b200 import report as RP


@pytest.mark.parametrize("x,want", [
    (1e-9, "1e-09"), (0.001, "0.001"), (0.0001, "0.0001"), (1e-5, "1e-05"), (1.5e-5, "1.5e-05"),
    (123.0, "123.0"), (0.99, "0.99"), (600.25, "600.25"), (1e15, "1e+15"), (123456789012345.0, "123456789012345.0"),
    (0.1, "0.1"), (2.5e-3, "0.0025"), (-3.75, "-3.75"), (0.0, "0.0"), (1e300, "1e+300"), (5e-324, "5e-324"),
    (0.30000000000000004, "0.30000000000000004"), (float("nan"), "null"),
])
def test_float_format(x, want):
    # nlohmann::json's number layout (shortest digits; fixed for exponents in (-4, 15])
    assert RP.format_float(x) == want


def test_serialize_layout_and_round_trip():
    cfg = rsm.RsmConfig(rank=3, mode=rsm.Mode.M2, plan=rsm.TrialPlan(600), seed=4)
    rep = rsm.DecompositionReport(e=0.0012345, trials_attempted=700, trials_accepted=600, z=41000,
                                  underdetermined_rows=2, gram_rank=197, borderline_rank_gate=False,
                                  wall_time=0.25)
    r = RP.make_report(cfg, rep, 1234567890123456789)
    assert r.block == 4 and r.trial_source == "explicit" and r.version == "0.1.0"
    text = RP.serialize_report(r)
    want = """{
  "version": "0.1.0",
  "dataset_checksum": 1234567890123456789,
  "seed": 4,
  "config": {
    "rank": 3,
    "mode": "m2",
    "block": 4,
    "vectors_per_trial": 0,
    "trials": 600,
    "trial_source": "explicit",
    "epsilon": 0.99,
    "workers": 0,
    "gram_rank_tol": 1e-09
  },
  "e": 0.0012345,
  "trials_attempted": 700,
  "trials_accepted": 600,
  "z": 41000,
  "underdetermined_rows": 2,
  "gram_rank": 197,
  "borderline_rank_gate": false,
  "wall_time": 0.25
}
"""
    assert text == want
    back = RP.parse_report(text)
    assert back == r
    assert RP.serialize_report(back) == text


def test_parse_errors():
    for bad in ["{", "[]", '{"version": "0.1.0"}']:
        with pytest.raises(rsm.Error) as ei:
            RP.parse_report(bad)
        assert ei.value.code == rsm.errc.parse_io
