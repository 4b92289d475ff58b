"""Run report: the reference's provenance record for one decompose run
(rsm::RunReport / make_report / serialize_report / parse_report,
include/rsm/io.hpp:25-45 and src/io.cpp:156-253 of /root/reference/proj),
so CLI-level reproducibility checks (tests/test_cli.cpp:78-105) can run
against this library.

serialize_report writes the layout the reference's
``nlohmann::ordered_json::dump(2) + "\\n"`` produces: keys in insertion order,
two-space indent, ``": "`` and ``",\\n"`` separators, and numbers in
nlohmann's float format -- the shortest round-trip digits, fixed notation
for decimal exponents in (-4, 15], otherwise ``d.ddde[+-]XX`` with at least
two exponent digits, and ``.0`` on integral values (see ``format_float``).
"""
from __future__ import annotations

import json
import math
from dataclasses import dataclass, field

from .rsm import DecompositionReport, Error, Mode, RsmConfig, errc

VERSION = "0.1.0"  # include/rsm/version.hpp:4


@dataclass
class RunReport:
    """rsm::RunReport (include/rsm/io.hpp:25-39)."""

    result: DecompositionReport = field(default_factory=DecompositionReport)
    rank: int = 0
    mode: Mode = Mode.M1
    block: int = 0
    vectors_per_trial: int = 0
    trials: int = 0
    trial_source: str = ""
    epsilon: float = 0.0
    seed: int = 0
    workers: int = 0
    gram_rank_tol: float = 0.0
    checksum: int = 0
    version: str = ""


def make_report(cfg: RsmConfig, rep: DecompositionReport, checksum: int) -> RunReport:
    """rsm::make_report (io.cpp:176-192): block 0 means the default r + 1."""
    return RunReport(result=rep, rank=cfg.rank, mode=Mode(cfg.mode),
                     block=cfg.block if cfg.block > 0 else cfg.rank + 1,
                     vectors_per_trial=cfg.vectors_per_trial, trials=cfg.plan.trials,
                     trial_source=cfg.plan.source, epsilon=cfg.plan.epsilon, seed=cfg.seed,
                     workers=cfg.workers, gram_rank_tol=cfg.gram_rank_tol, checksum=checksum,
                     version=VERSION)


def format_float(x: float) -> str:
    """A double as nlohmann::json prints it (shortest round trip, Grisu-style
    layout with kMinExp = -4, kMaxExp = 15)."""
    if not math.isfinite(x):
        return "null"
    if x == 0.0:
        return "-0.0" if math.copysign(1.0, x) < 0 else "0.0"
    sign = "-" if x < 0 else ""
    mant, _, exp = repr(abs(x)).partition("e")
    ip, _, fp = mant.partition(".")
    digits = (ip + fp).lstrip("0")
    # value = 0.digits... placed so that n digits precede the decimal point
    n = len(ip.lstrip("0")) if ip.strip("0") else -(len(fp) - len(fp.lstrip("0")))
    n += int(exp) if exp else 0
    digits = digits.rstrip("0") or "0"
    k = len(digits)
    if k <= n <= 15:
        return sign + digits + "0" * (n - k) + ".0"
    if 0 < n <= 15:
        return sign + digits[:n] + "." + digits[n:]
    if -4 < n <= 0:
        return sign + "0." + "0" * (-n) + digits
    e = n - 1
    es = ("-" if e < 0 else "+") + ("%02d" % abs(e))
    return sign + digits[0] + ("." + digits[1:] if k > 1 else "") + "e" + es


def _dump(obj, indent=0) -> str:
    pad = " " * (indent + 2)
    if isinstance(obj, dict):
        if not obj:
            return "{}"
        items = [pad + json.dumps(k) + ": " + _dump(v, indent + 2) for k, v in obj.items()]
        return "{\n" + ",\n".join(items) + "\n" + " " * indent + "}"
    if isinstance(obj, bool):
        return "true" if obj else "false"
    if isinstance(obj, int):
        return str(obj)
    if isinstance(obj, float):
        return format_float(obj)
    return json.dumps(obj)


def serialize_report(r: RunReport) -> str:
    """rsm::serialize_report (io.cpp:194-216)."""
    j = {
        "version": r.version,
        "dataset_checksum": int(r.checksum),
        "seed": int(r.seed),
        "config": {
            "rank": int(r.rank),
            "mode": "m1" if Mode(r.mode) == Mode.M1 else "m2",
            "block": int(r.block),
            "vectors_per_trial": int(r.vectors_per_trial),
            "trials": int(r.trials),
            "trial_source": r.trial_source,
            "epsilon": float(r.epsilon),
            "workers": int(r.workers),
            "gram_rank_tol": float(r.gram_rank_tol),
        },
        "e": float(r.result.e),
        "trials_attempted": int(r.result.trials_attempted),
        "trials_accepted": int(r.result.trials_accepted),
        "z": int(r.result.z),
        "underdetermined_rows": int(r.result.underdetermined_rows),
        "gram_rank": int(r.result.gram_rank),
        "borderline_rank_gate": bool(r.result.borderline_rank_gate),
        "wall_time": float(r.result.wall_time),
    }
    return _dump(j) + "\n"


def parse_report(text: str) -> RunReport:
    """rsm::parse_report (io.cpp:218-253); malformed input is errc::parse_io."""
    try:
        j = json.loads(text)
    except ValueError as e:
        raise Error(errc.parse_io, "bad report json: " + str(e))
    try:
        c = j["config"]
        res = DecompositionReport(e=float(j["e"]), trials_attempted=int(j["trials_attempted"]),
                                  trials_accepted=int(j["trials_accepted"]), z=int(j["z"]),
                                  underdetermined_rows=int(j["underdetermined_rows"]),
                                  gram_rank=int(j["gram_rank"]),
                                  borderline_rank_gate=bool(j["borderline_rank_gate"]),
                                  wall_time=float(j["wall_time"]))
        return RunReport(result=res, rank=int(c["rank"]), mode=Mode.M2 if c["mode"] == "m2" else Mode.M1,
                         block=int(c["block"]), vectors_per_trial=int(c["vectors_per_trial"]),
                         trials=int(c["trials"]), trial_source=str(c["trial_source"]),
                         epsilon=float(c["epsilon"]), seed=int(j["seed"]), workers=int(c["workers"]),
                         gram_rank_tol=float(c["gram_rank_tol"]), checksum=int(j["dataset_checksum"]),
                         version=str(j["version"]))
    except (KeyError, TypeError, ValueError) as e:
        raise Error(errc.parse_io, "bad report json: " + str(e))
