"""CPU: the loader path pinned to the REFERENCE'S OWN io.cpp (src/io.cpp:56-254
compiled into oracle/_ref by oracle/build_ref.sh against the image's nlohmann
JSON header): load_matrix, save_matrix, dataset_checksum, make_report +
serialize_report and parse_report, through the library's C-ABI and report.py.

Two layers: the committed fixtures tests/golden/io_ref.json (written by the
reference via tests/golden/make_golden_io.py) always; the live reference build
in addition when oracle/_ref has io.cpp (this container)."""
import json
import os

import numpy as np
import pytest

from oracle import refbind as R
from paper_1411_0814_b200 import report as RP
from paper_1411_0814_b200 import rsm
from tests.golden.make_golden_io import MATS, REPORTS, matrix
from tests.test_io_loader import CASES, ERRORS

GOLD = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "io_ref.json")))
live = pytest.mark.skipif(not R.have_io(), reason="oracle/_ref built without io.cpp (needs /root/reference)")


def _write(d, name, text):
    p = os.path.join(d, name + ".csv")
    with open(p, "wb") as f:
        f.write(text.encode())
    return p


@pytest.mark.parametrize("name", sorted(CASES))
def test_load_matches_reference_fixture(tmp_path, name):
    M = rsm.load_matrix(_write(str(tmp_path), name, CASES[name]))
    g = GOLD["loads"][name]
    assert [M.m, M.n] == g["shape"]
    assert M.mask.ravel().tolist() == g["mask"]
    assert [int(x) for x in M.values.ravel().view(np.uint64)] == [int(x) for x in g["bits"]]


@pytest.mark.parametrize("name", sorted(ERRORS))
def test_load_errors_match_reference_fixture(tmp_path, name):
    with pytest.raises(rsm.Error) as ei:
        rsm.load_matrix(_write(str(tmp_path), name, ERRORS[name][0]))
    assert int(ei.value.code) == GOLD["load_errors"][name] == int(rsm.errc.parse_io)


@pytest.mark.parametrize("i", range(len(MATS)))
def test_save_text_and_checksum_match_reference_fixture(tmp_path, i):
    m, n, rho, seed, spread = MATS[i]
    Y, W = matrix(m, n, rho, seed, spread)
    M = rsm.MaskedMatrix(m, n, Y, W)
    p = os.path.join(str(tmp_path), "s.csv")
    rsm.save_matrix(M, p)
    assert open(p, "rb").read().decode() == GOLD["mats"][i]["text"]
    assert rsm.dataset_checksum(M) == int(GOLD["mats"][i]["checksum"])


def _our_report(f):
    rank, mode, block, vpt, trials, eps, seed, tol, workers, e, att, acc, z, und, grank, border, wall, chk = f
    cfg = rsm.RsmConfig(rank=rank, mode=rsm.Mode.M2 if mode else rsm.Mode.M1, block=block, vectors_per_trial=vpt,
                        plan=rsm.TrialPlan(trials, epsilon=eps), seed=seed, gram_rank_tol=tol, workers=workers)
    rep = rsm.DecompositionReport(e=e, trials_attempted=att, trials_accepted=acc, z=z, underdetermined_rows=und,
                                  gram_rank=grank, borderline_rank_gate=border, wall_time=wall)
    return RP.serialize_report(RP.make_report(cfg, rep, chk))


@pytest.mark.parametrize("i", range(len(REPORTS)))
def test_report_text_matches_reference_fixture(i):
    text = _our_report(REPORTS[i])
    assert text == GOLD["reports"][i]["text"]
    # parse -> serialize round trip agrees with the reference's
    assert RP.serialize_report(RP.parse_report(text)) == GOLD["reports"][i]["reparsed"]


@live
def test_live_reference_loads_saves_and_checksums(tmp_path):
    d = str(tmp_path)
    for name, text in CASES.items():
        p = _write(d, name, text)
        Y, W = R.load_matrix(p)
        M = rsm.load_matrix(p)
        assert np.array_equal(M.mask, W)
        assert np.array_equal(M.values.view(np.uint64)[W == 1], Y.view(np.uint64)[W == 1])
    rng = np.random.default_rng(3)
    for t in range(20):
        m, n = int(rng.integers(1, 40)), int(rng.integers(1, 40))
        Y, W = matrix(m, n, float(rng.uniform(0.05, 1.0)), 1000 + t, float(rng.uniform(0, 30)))
        M = rsm.MaskedMatrix(m, n, Y, W)
        assert rsm.dataset_checksum(M) == R.dataset_checksum(Y, W)
        p1, p2 = os.path.join(d, "a.csv"), os.path.join(d, "b.csv")
        rsm.save_matrix(M, p1)
        R.save_matrix(Y, W, p2)
        assert open(p1, "rb").read() == open(p2, "rb").read()


@live
def test_live_reference_reports():
    rng = np.random.default_rng(9)
    for t in range(50):
        e = float(10.0 ** rng.uniform(-300, 300)) * float(rng.choice([1, -1]))
        wall = float(rng.uniform(0, 1e4))
        f = (int(rng.integers(1, 9)), int(rng.integers(0, 2)), int(rng.integers(0, 12)), int(rng.integers(0, 3)),
             int(rng.integers(1, 2**40)), float(rng.uniform(0.5, 0.999)), int(rng.integers(0, 2**63)),
             float(10.0 ** rng.uniform(-15, -3)), int(rng.integers(0, 64)), e, int(rng.integers(0, 2**50)),
             int(rng.integers(0, 2**40)), int(rng.integers(0, 2**60)), int(rng.integers(0, 2**30)),
             int(rng.integers(0, 5000)), bool(rng.integers(0, 2)), wall, int(rng.integers(0, 2**63)))
        assert _our_report(f) == R.serialize_report(*f)
