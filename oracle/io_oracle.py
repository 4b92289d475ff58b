"""Test infrastructure only: a pure-Python restatement of the reference's
NaN-CSV loader/saver and dataset checksum (src/io.cpp:17-154 of
/root/reference/proj), the checker for rsm_load_matrix_csv /
rsm_save_matrix_csv / rsm_dataset_checksum. The reference's io.cpp is not in
oracle/_ref (it needs the absent nlohmann json.hpp), so this restatement is
pinned by the reference's own test_io.cpp cases, restated in
tests/test_io_loader.py. Returns (values, mask) numpy arrays or raises
IoOracleError(code, message) with the reference's codes (3 = parse_io,
2 = invalid_config) and messages.
"""
import math
import struct

import numpy as np


class IoOracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code
        self.msg = msg


_WS = " \t\n\v\f\r"  # std::isspace in the C locale


def _lines(text):
    """std::getline over a binary stream, with io.cpp:63-64's '\\r' strip and
    trailing-empty-line break."""
    out = []
    pos, N = 0, len(text)
    while pos < N:
        eol = text.find("\n", pos)
        last = eol < 0
        if last:
            eol = N
        line = text[pos:eol]
        if line.endswith("\r"):
            line = line[:-1]
        if line == "" and (last or eol + 1 >= N):  # in.peek() == EOF
            break
        out.append(line)
        if last:
            break
        pos = eol + 1
    return out


def _strtod_full(tok):
    """strtod must consume the whole token and give a finite value."""
    body = tok.lstrip("+-")
    try:
        if body[:2].lower() == "0x":  # strtod's hexadecimal form
            v = float.fromhex(tok)
        else:
            v = float(tok)
    except ValueError:
        return None
    # float() accepts forms strtod rejects or vice versa only at the margins
    # ('1_0', 'infinity'); those fail either way below or are not finite
    if "_" in tok or not math.isfinite(v):
        return None
    return v


def load_matrix(path):
    try:
        with open(path, "rb") as f:
            text = f.read().decode("latin-1")
    except OSError:
        raise IoOracleError(3, "cannot open file: " + path)
    rows, width = [], 0
    for line in _lines(text):
        row = []
        for raw in line.split(","):
            cell = raw.strip(_WS)
            if cell == "" or (len(cell) == 3 and cell.lower() == "nan"):
                row.append(None)
                continue
            v = _strtod_full(cell)
            if v is None:
                raise IoOracleError(3, "non-numeric token '" + cell + "' in " + path)
            row.append(v)
        if width == 0:
            width = len(row)
        if len(row) != width:
            raise IoOracleError(3, "ragged row " + str(len(rows) + 1) + " in " + path)
        rows.append(row)
    if not rows or width == 0:
        raise IoOracleError(3, "empty matrix in " + path)
    m, n = len(rows), width
    Y = np.full((m, n), np.nan)
    W = np.zeros((m, n), np.uint8)
    for i, row in enumerate(rows):
        for j, v in enumerate(row):
            if v is not None:
                Y[i, j], W[i, j] = v, 1
    return Y, W


def save_text(Y, W):
    """The text save_matrix writes (io.cpp:101-116)."""
    m, n = Y.shape
    if m < 1 or n < 1:
        raise IoOracleError(2, "cannot save an empty matrix")
    lines = []
    for i in range(m):
        cells = [("%.17g" % Y[i, j]) if W[i, j] else "NaN" for j in range(n)]
        lines.append(",".join(cells) + "\n")
    return "".join(lines)


def dataset_checksum(Y, W):
    """FNV-1a 64 over dims, then known byte + value bits per cell (io.cpp:131-154)."""
    h = 0xcbf29ce484222325
    M64 = (1 << 64) - 1

    def feed(b):
        nonlocal h
        for x in b:
            h ^= x
            h = (h * 0x100000001b3) & M64

    m, n = W.shape
    feed(struct.pack("<QQ", m, n))
    for q, k in enumerate(W.reshape(-1)):
        feed(bytes([1 if k else 0]))
        if k:
            feed(struct.pack("<d", float(Y.reshape(-1)[q])))
    return h
