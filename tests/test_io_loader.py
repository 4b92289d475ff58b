"""CPU: the loader path -- NaN-CSV load/save
and the dataset checksum of the library (host C++ behind the C-ABI) against
oracle/io_oracle.py (a restatement of src/io.cpp:17-154), with the cases of
the reference's own tests/test_io.cpp restated; and the config-5 track
generator against its C restatement in oracle/rsm_oracle.c."""
import os

import numpy as np
import pytest

from oracle import io_oracle as IO
from oracle import oracle as O
from paper_1411_0814_b200 import rsm
from tests.util import random_masked

CASES = {  # name -> file text
    "basic": "1,2\n3,NaN\n",
    "tokens": "1,,3\nnan,NAN,2.5e-3\n",
    "crlf": " 1 , 2 \r\n 3 , 4 \r\n",
    "no_final_newline": "1,2\n3,4",
    "extra_blank_line": "1,2\n3,4\n\n",
    "cr_only_last": "5,6\n\r",
    "spaces_nan": " nan ,\t7 \n8, NaN \n",
    "exp_forms": "1e-300,-2.5E+10\n0x1p-3,.5\n",
    "single_col": "1\n\n2\n",
}
ERRORS = {  # name -> (text, message prefix)
    "ragged": ("1,2\n3\n", "ragged row 2 in "),
    "junk": ("1,abc\n", "non-numeric token 'abc' in "),
    "inf": ("1,inf\n", "non-numeric token 'inf' in "),
    "empty": ("", "empty matrix in "),
    "blank_middle": ("1,2\n\n3,4\n", "ragged row 2 in "),
    "nan4": ("nann,1\n", "non-numeric token 'nann' in "),
}


def _write(tmp_path, name, text):
    p = os.path.join(tmp_path, name + ".csv")
    with open(p, "wb") as f:
        f.write(text.encode())
    return p


@pytest.mark.parametrize("name", sorted(CASES))
def test_load_matches_restatement(tmp_path, name):
    p = _write(str(tmp_path), name, CASES[name])
    M = rsm.load_matrix(p)
    Y, W = IO.load_matrix(p)
    assert (M.m, M.n) == Y.shape
    assert np.array_equal(M.mask, W)
    k = W.astype(bool)
    assert np.array_equal(M.values[k].view(np.uint64), Y[k].view(np.uint64))
    assert np.isnan(M.values[~k]).all()


def test_reference_io_cases(tmp_path):
    # tests/test_io.cpp:24-57 of the reference, restated
    M = rsm.load_matrix(_write(str(tmp_path), "b", "1,2\n3,NaN\n"))
    assert (M.m, M.n) == (2, 2) and M.values[0, 0] == 1 and M.values[0, 1] == 2 and M.values[1, 0] == 3
    assert M.mask.tolist() == [[1, 1], [1, 0]]
    M = rsm.load_matrix(_write(str(tmp_path), "t", "1,,3\nnan,NAN,2.5e-3\n"))
    assert M.known_count() == 3 and M.values[1, 2] == 2.5e-3
    M = rsm.load_matrix(_write(str(tmp_path), "c", " 1 , 2 \r\n 3 , 4 \r\n"))
    assert M.m == 2 and M.values[1, 1] == 4.0 and M.known_count() == 4


@pytest.mark.parametrize("name", sorted(ERRORS))
def test_load_errors(tmp_path, name):
    text, msg = ERRORS[name]
    p = _write(str(tmp_path), name, text)
    with pytest.raises(rsm.Error) as ei:
        rsm.load_matrix(p)
    with pytest.raises(IO.IoOracleError) as eo:
        IO.load_matrix(p)
    assert ei.value.code == rsm.errc.parse_io == eo.value.code
    assert str(ei.value).endswith(msg + p) or (msg + p) in str(ei.value)
    assert eo.value.msg == msg + p


def test_missing_file_is_parse_io():
    with pytest.raises(rsm.Error) as ei:
        rsm.load_matrix("no_such_file_anywhere.csv")
    assert ei.value.code == rsm.errc.parse_io
    assert "cannot open file: no_such_file_anywhere.csv" in str(ei.value)


def test_save_text_and_round_trip_bit_exact(tmp_path):
    # tests/test_io.cpp:83-95: save then load is bit-exact; the text matches
    # the restatement byte for byte
    Y, W = random_masked(23, 17, 0.7, 13)
    Y = Y * np.exp(np.random.default_rng(5).standard_normal(Y.shape) * 20)  # wide exponent range
    M = rsm.MaskedMatrix(23, 17, np.where(W.astype(bool), Y, np.nan), W)
    p = os.path.join(str(tmp_path), "rt.csv")
    rsm.save_matrix(M, p)
    with open(p, "rb") as f:
        assert f.read().decode() == IO.save_text(M.values, M.mask)
    R = rsm.load_matrix(p)
    assert np.array_equal(R.mask, M.mask)
    k = M.mask.astype(bool)
    assert np.array_equal(R.values[k].view(np.uint64), M.values[k].view(np.uint64))


def test_save_empty_is_invalid_config(tmp_path):
    with pytest.raises(rsm.Error) as ei:
        rsm.lib()  # loaded
        st = rsm.lib().rsm_save_matrix_csv(os.fsencode(os.path.join(str(tmp_path), "x.csv")), None, None, 0, 3)
        raise rsm.Error(st, "")
    assert ei.value.code == rsm.errc.invalid_config


def test_checksum_matches_restatement_and_reference_properties():
    # tests/test_io.cpp:108-142: stable, value- and mask-sensitive, blind to hidden cells
    Y, W = random_masked(12, 9, 0.6, 19)
    M = rsm.MaskedMatrix(12, 9, Y, W)
    h = rsm.dataset_checksum(M)
    assert h == IO.dataset_checksum(M.values, M.mask) == rsm.dataset_checksum(M)
    i, j = np.argwhere(W == 1)[0]
    bumped = rsm.MaskedMatrix(12, 9, M.values.copy(), W.copy())
    bumped.values[i, j] = np.nextafter(bumped.values[i, j], np.inf)
    assert rsm.dataset_checksum(bumped) != h
    i, j = np.argwhere(W == 0)[0]
    poked = rsm.MaskedMatrix(12, 9, M.values.copy(), W.copy())
    poked.values[i, j] = 123.0
    assert rsm.dataset_checksum(poked) == h
    remasked = rsm.MaskedMatrix(12, 9, M.values.copy(), W.copy())
    remasked.mask[i, j] = 1
    remasked.values[i, j] = 0.0
    assert rsm.dataset_checksum(remasked) != h


@pytest.mark.parametrize("case", [(300, 64, 8, 32, 1e-3, 3), (97, 40, 40, 40, 0.0, 5), (50, 10, 1, 10, 0.1, 0)])
def test_track_generator_matches_restatement(case):
    pts, frames, wmin, wmax, sigma, seed = case
    M = rsm.generate_tracks(pts, frames, wmin, wmax, sigma, seed)
    Y, W = O.generate_tracks(pts, frames, wmin, wmax, sigma, seed)
    assert np.array_equal(M.mask, W)
    k = W.astype(bool)
    assert np.array_equal(M.values[k].view(np.uint64), Y[k].view(np.uint64))
    # row blocks are independent of the split
    part = rsm.generate_tracks(pts, frames, wmin, wmax, sigma, seed, row0=7, rows=20)
    assert np.array_equal(part.mask, W[7:27])


def test_track_generator_structure():
    pts, frames, wmin, wmax = 400, 128, 16, 64
    M = rsm.generate_tracks(pts, frames, wmin, wmax, 0.0, 11)
    W = M.mask.reshape(pts, frames, 2)
    assert (W[:, :, 0] == W[:, :, 1]).all()  # both coordinates of a frame together
    for i in range(pts):
        vis = np.flatnonzero(W[i, :, 0])
        assert wmin <= len(vis) <= wmax and vis[-1] - vis[0] + 1 == len(vis)  # one contiguous window
    # noiseless: every fully observed block has rank 4 (points x affine cameras)
    rows = np.flatnonzero(W[:, 40:48, 0].all(axis=1))
    blk = M.values[np.ix_(rows, np.arange(80, 96))]
    sv = np.linalg.svd(blk, compute_uv=False)
    assert len(rows) >= 8 and sv[4] <= 1e-12 * sv[0] and sv[3] > 1e-6 * sv[0]


def test_track_generator_validation():
    for args in [(0, 10, 1, 5), (10, 10, 0, 5), (10, 10, 6, 5), (10, 10, 1, 11)]:
        with pytest.raises(rsm.Error):
            rsm.generate_tracks(*args, 0.0, 0)
