#!/usr/bin/env python
"""Benchmark of the B200 RSM hot path (driver contract).

Workload (config.workload): BASELINE.json config 3, "the paper's synthetic
scale": m=131072, n=1024, r=4, rho=0.8, sigma=1e-3, row branch k=5, 16384
submatrices, seed 0 (BASELINE.json gives none; 0 documented). A step is one
full RSM decomposition (selection, SVD, Gram, eigen-extraction, U solve, e).
The input is synthetic, generated on the host from the reference generator's
streams (src/synth.cpp:12-57); no public dataset is involved.

  value   submatrices/s of the whole job = T / device time of one decompose,
          with Y and the mask already resident in HBM; CUDA events on the
          library's stream; L2 flushed (256 MiB write) between steps, untimed.
  e2e     the same metric through the public API with host buffers: pinned
          H2D of Y (FP64) + mask (uint8), decompose, D2H of U and V, per step.
  roofline for the dominant kernel; stages{} gives every stage's share.
  cpu_baseline  the reference CPU path (oracle/_ref: the reference's own
          sources) on a bounded sample of the same workload, extrapolated.

--impl reference runs the reference's CPU implementation alone (rank 0).
Multi-GPU (torchrun): trials shard over ranks inside one decomposition with a
single NCCL all-reduce of the n x n accumulator, Y rows shard for the U solve
(strong scaling: the total work is one decomposition of config 3).
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CFG = dict(workload="config3_row_branch_131072x1024_r4", m=131072, n=1024, r=4, rho=0.8, sigma=1e-3, k=5,
           T=16384, seed=0)
CONFIGS = {
    "config3": CFG,
    "config1": dict(workload="config1_row_branch_2000x200_r3", m=2000, n=200, r=3, rho=0.8, sigma=1e-3, k=4,
                    T=2000, seed=0),
    "config4": dict(workload="config4_row_branch_1048576x2048_r8", m=1048576, n=2048, r=8, rho=0.9, sigma=1e-3,
                    k=9, T=65536, seed=0),
}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("hbm_gbs", 6650.0), "measured"
    return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.p = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}.csv")

    def start(self):
        try:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            self.f = open(self.path, "w")
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-i", str(self.index), "-lms", "200"], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        out = {"sm_mhz": None, "sm_max_mhz": None, "reasons": []}
        if self.p is None:
            return out
        time.sleep(0.25)
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.close()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if sm:
            load = [s for s in sm if s > 0.5 * max(sm)] or sm
            out = {"sm_mhz": statistics.median(load), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                   "samples": len(sm)}
        return out


def gen_input(c, rank=0):
    from paper_1411_0814_b200 import rsm
    import torch
    m, n = c["m"], c["n"]
    # pinned host buffers for the e2e leg (H2D from pinned memory)
    Yt = torch.empty((m, n), dtype=torch.float64, pin_memory=True)
    Wt = torch.empty((m, n), dtype=torch.uint8, pin_memory=True)
    Y, W = Yt.numpy(), Wt.numpy()
    block = 65536
    for r0 in range(0, m, block):
        rows = min(block, m - r0)
        st = rsm.lib().rsm_generate(m, n, c["r"], c["rho"], c["sigma"], c["seed"], r0, rows,
                                    Y[r0:r0 + rows].ctypes.data_as(rsm.C.c_void_p),
                                    W[r0:r0 + rows].ctypes.data_as(rsm.C.c_void_p))
        assert st == 0
    return Yt, Wt, Y, W


def algorithmic(c, qs, nwp_bytes, attempts):
    """Algorithmic work per stage."""
    m, n, r, k, T = c["m"], c["n"], c["r"], c["k"], c["T"]
    q = qs.astype(np.float64)
    s1_bytes = attempts * k * (n / 32) * 4                           # selection: drawn rows' mask words
    s2_bytes = T * k * n * 8                                         # gather: full Y rows (SURVEY 8d S1 note)
    s2_flops = float(np.sum(2 * q * k * (k + 1) / 2 + 2 * r * k * q))
    s3_flops = float(np.sum(r * q * (q + 1)))                        # symmetric rank-r updates (unique entries)
    s3_flops_survey = float(np.sum(2 * r * q * q))                   # SURVEY 8d literal-symmetric count
    s4_bytes = n * n * 8
    s5_bytes = m * n * 8 + m * nwp_bytes + m * r * 8 + n * r * 8
    return dict(s1_bytes=s1_bytes, s2_bytes=s2_bytes, s2_flops=s2_flops, s3_flops=s3_flops, s3_flops_survey=s3_flops_survey,
                s4_bytes=s4_bytes, s5_bytes=s5_bytes)


# ------------------------------------------------------------------ CPU arm

def cpu_reference_sample(Y, W, c, G=None, V=None, trials_prefix=64, rows_sample=16384):
    """Time the reference CPU path (oracle/_ref: the reference's own sources,
    all host threads) on a bounded sample of the workload and extrapolate one
    full decomposition:
      harvest_gram on the first `trials_prefix` accepted trials (per-trial work
        is i.i.d., so the full harvest is that time x T / accepted);
      solve_v (LAPACKE dsyev + rank gate) on G -- the full accumulator when the
        caller has it, else the reference's own prefix accumulator (same n x n
        dsyev; its rank gate may fail on a prefix, after dsyev has run);
      solve_u + the e pass on `rows_sample` rows against V (the decomposition's
        V-hat, else the planted basis it converges to), x m / rows.
    Every factor is returned as a field."""
    from oracle import refbind as R
    if not R.available():
        return None
    threads = os.cpu_count() or 1
    os.environ.setdefault("OMP_NUM_THREADS", str(threads))
    m, n, r = c["m"], c["n"], c["r"]

    class P:
        pass
    p = P()
    p.mode, p.block, p.rank, p.min_count, p.seed, p.ell = 1, c["k"], r, r + 1, c["seed"], 0
    Gp, att, acc, _, t_h = R.harvest(Y, W, p, trials_prefix, workers=threads, timed=True)
    g_src = "full accumulator (device harvest)" if G is not None else f"reference prefix accumulator ({acc} trials)"
    Vv, gr, _, t_v = R.solve_v(G if G is not None else Gp, r, 1e-9, timed=True, gate_failure_ok=True)
    if V is None:
        V = Vv
    v_src = "V-hat of the decomposition"
    if V is None:
        _, _, B = R.generate(min(m, 2 * n), n, r, c["rho"], c["sigma"], c["seed"], with_basis=True)
        V = np.linalg.qr(B)[0]
        v_src = "planted basis (orthonormalised)"
    rs = min(rows_sample, m)
    Ys, Ws = np.ascontiguousarray(Y[:rs]), np.ascontiguousarray(W[:rs])
    _, _, t_u = R.solve_u(Ys, Ws, np.ascontiguousarray(V), r, workers=threads, timed=True)
    f_h, f_u = c["T"] / max(acc, 1), m / rs
    est = t_h * f_h + t_v + t_u * f_u
    sample = (f"harvest_gram on the first {acc} accepted trials ({t_h:.2f}s, x{f_h:.0f}), solve_v dsyev(n={n}) on "
              f"the {g_src} ({t_v:.2f}s), solve_u+residual on {rs} rows against the {v_src} ({t_u:.2f}s, "
              f"x{f_u:.0f}); extrapolated full decompose {est:.1f}s")
    return dict(value=c["T"] / est, unit="submatrices/s", cores=threads, kind="reference", sample=sample,
                est_decompose_s=est, sample_s=t_h + t_v + t_u,
                extrapolation={"harvest_s": t_h, "harvest_trials": acc, "harvest_factor": f_h, "solve_v_s": t_v,
                               "solve_v_input": g_src, "solve_u_s": t_u, "solve_u_rows": rs, "solve_u_factor": f_u,
                               "solve_u_basis": v_src})


def cpu_reference_config1(threads=None):
    """A fully measured (not extrapolated) reference decomposition of BASELINE
    config 1 (2000 x 200, r = 3, k = 4, 2000 submatrices): the reference's own
    rsm::decompose on its own generator's instance."""
    from oracle import refbind as R
    if not R.available():
        return None
    c = CONFIGS["config1"]
    threads = threads or os.cpu_count() or 1
    Y, W = R.generate(c["m"], c["n"], c["r"], c["rho"], c["sigma"], c["seed"])
    t0 = time.perf_counter()
    out = R.decompose(Y, W, c["r"], c["T"], mode=1, block=c["k"], seed=c["seed"], workers=threads)
    wall = time.perf_counter() - t0
    return {"workload": c["workload"], "decompose_s": wall, "value": c["T"] / wall, "unit": "submatrices/s",
            "cores": threads, "e": out[2]["e"], "measured": "full decompose, not extrapolated"}


def arm_config(c, world):
    """The `config` object both arms print (same workload, same keys)."""
    return {"workload": c["workload"], "m": c["m"], "n": c["n"], "r": c["r"], "rho": c["rho"], "sigma": c["sigma"],
            "k": c["k"], "trials": c["T"], "seed": c["seed"], "parallelism": f"trials+rows x{world}",
            "l2": f"flushed (256 MiB write) between timed steps; Y ({c['m'] * c['n'] * 8 / 2**30:.2f} GiB) vs 126 MB L2"}


def run_reference_arm(args, c):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import refbind as R
    if not R.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built (needs /root/reference)"}))
        return 0
    m, n = c["m"], c["n"]
    # the reference's own generator (src/synth.cpp via oracle/_ref), not ours
    Y, W = R.generate(m, n, c["r"], c["rho"], c["sigma"], c["seed"])
    vals = []
    for s in range(args.warmup + args.steps):
        # >= 4 trials per host thread, so the prefix keeps every thread busy
        res = cpu_reference_sample(Y, W, c, trials_prefix=max(32, 4 * (os.cpu_count() or 1)), rows_sample=4096)
        if s >= args.warmup:
            vals.append(res)
    v = statistics.median([x["value"] for x in vals])
    est = statistics.median([x["est_decompose_s"] for x in vals])
    step_s = statistics.median([x["sample_s"] for x in vals])  # what one step actually ran (the bounded sample)
    c1 = cpu_reference_config1()
    line = {"metric": "submatrices/s (full RSM decompose)", "value": v, "unit": "submatrices/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_s * 1e3,
            "est_decompose_ms": est * 1e3,
            "ms_per_step_note": "one step = the bounded sample in cpu_baseline.sample (measured); value = T / the "
                                "full decomposition extrapolated from it (est_decompose_ms, factors in "
                                "cpu_baseline.extrapolation)",
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference generator streams, seed 0)",
            "config": arm_config(c, args.gpus),
            "impl": "reference",
            "cpu_baseline": {"value": v, "unit": "submatrices/s", "cores": vals[0]["cores"], "kind": "reference",
                             "sample": vals[0]["sample"], "extrapolation": vals[len(vals) // 2]["extrapolation"]},
            "e2e": {"value": v, "unit": "submatrices/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "config1_measured": c1}
    print(json.dumps(line))
    return 0


# ------------------------------------------------------------------ GPU arm

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="config3", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--stages", action="store_true", help="print per-stage ms to stderr")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    c = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference_arm(args, c)

    import torch
    from paper_1411_0814_b200 import rsm
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    nccl_id = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        obj = [rsm.Context.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    ctx = rsm.Context(local, world, rank, nccl_id)
    m, n, r, T = c["m"], c["n"], c["r"], c["T"]
    # a large instance (config 4: 16 GiB of values) is generated on each rank's
    # device for the resident leg; the host copy the e2e leg uploads is pinned
    # per rank only while all ranks together stay within HOST_PIN_BUDGET
    host_bytes = m * n * 9
    big = host_bytes > (4 << 30)
    host_ok = host_bytes * world <= int(os.environ.get("HOST_PIN_BUDGET", str(96 << 30)))
    Yt = Wt = Y = W = None
    if host_ok:
        Yt, Wt, Y, W = gen_input(c, rank)
    cfg = rsm.RsmConfig(rank=r, mode=rsm.Mode.M2, block=c["k"], plan=rsm.TrialPlan(T), seed=c["seed"])
    stream = torch.cuda.ExternalStream(ctx.stream)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{local}")

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()

    # ---- device-resident leg (value) ----
    if big or Y is None:
        ctx.generate(m, n, r, c["rho"], c["sigma"], c["seed"])  # the same instance, on the device
    else:
        ctx.load_arrays(Y, W)
    for _ in range(args.warmup):
        ctx.decompose(cfg, fetch=False)
    clocks = Clocks(local)
    barrier()
    clocks.start()
    times, stage_rows, launches = [], [], 0
    for _ in range(args.steps):
        flush.zero_()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        _, rep = ctx.decompose(cfg, fetch=False)
        e1.record(stream)
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
        stage_rows.append(ctx.stage_ms())
        launches += ctx.launch_count()
    barrier()
    clk = clocks.stop()
    tot = torch.tensor([sum(times)], dtype=torch.float64, device=f"cuda:{local}")
    if dist is not None:
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    ms_per_step = tot.item() / args.steps
    value = T / (ms_per_step / 1e3)

    # ---- end-to-end leg (public API, host buffers) ----
    e2e_times = []
    for s in range(args.warmup + args.steps if host_ok else 0):
        flush.zero_()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        ctx.load_arrays(Y, W)
        F, rep2 = ctx.decompose(cfg, fetch=True)
        e1.record(stream)
        e1.synchronize()
        if s >= args.warmup:
            e2e_times.append(e0.elapsed_time(e1))
    et = torch.tensor([sum(e2e_times)], dtype=torch.float64, device=f"cuda:{local}")
    if dist is not None:
        dist.all_reduce(et, op=dist.ReduceOp.MAX)
    e2e_ms = et.item() / args.steps
    h2d = ctx.last_load_h2d_bytes() if host_ok else 0  # values + the mask as bit-packed on the host
    d2h = (m + n) * r * 8 if host_ok else 0

    # ---- roofline of the dominant kernel ----
    st = np.array(stage_rows)  # select, svd, gram, reduce, solve_v, solve_u, total
    med = np.median(st, axis=0)
    names = ["select", "svd", "gram", "gram_reduce", "solve_v", "solve_u"]
    ids, qs, att, acc = ctx.select(rsm.TrialParams(rsm.Mode.M2, c["k"], 0, r, r + 1, c["seed"]), T)
    alg = algorithmic(c, qs, ((n + 127) // 128) * 4 * 4, att)
    hbm, hbm_src = peaks()
    fp64 = rsm.fp64_peak_tflops(local)
    stage_info = {}
    for i, nm in enumerate(names):
        stage_info[nm] = {"ms": float(med[i]), "share": float(med[i] / med[6]) if med[6] > 0 else None}
    stage_info["select"].update(alg_bytes=alg["s1_bytes"], gbs=alg["s1_bytes"] / (med[0] * 1e-3) / 1e9)
    stage_info["svd"].update(alg_flops=alg["s2_flops"], tflops=alg["s2_flops"] / (med[1] * 1e-3) / 1e12,
                             alg_bytes=alg["s2_bytes"], gbs=alg["s2_bytes"] / (med[1] * 1e-3) / 1e9)
    # SURVEY.md 8(d) S3 count, 2 r q^2 per trial (the roofline figure); the
    # unique-entry count r q (q + 1) of the symmetric update is reported beside it
    stage_info["gram"].update(alg_flops=alg["s3_flops_survey"],
                              tflops=alg["s3_flops_survey"] / (med[2] * 1e-3) / 1e12,
                              alg_flops_unique=alg["s3_flops"],
                              tflops_unique=alg["s3_flops"] / (med[2] * 1e-3) / 1e12)
    stage_info["solve_v"].update(alg_bytes=alg["s4_bytes"])
    stage_info["solve_u"].update(alg_bytes=alg["s5_bytes"], gbs=alg["s5_bytes"] / (med[5] * 1e-3) / 1e9)
    dom = names[int(np.argmax(med[:6]))]
    if dom == "gram" and os.environ.get("RSM_GRAM", "") != "dfma":
        # stage 3 runs on the tcgen05 tensor cores as an exact int8 digit
        # split (k_gram_i8.cu): bound = the int8 tensor pipe. achieved = the
        # int8 MMA operations the kernel's algorithm issues (upper-triangle
        # 128 x 64 tiles x K = trials * r rows x S(S+1)/2 digit pairs x 2);
        # the FP64 work it stands for is reported beside it
        # against the FP64 (DFMA) peak.
        S = int(os.environ.get("RSM_I8_SLICES", "6"))
        npad = ((n + 127) // 128) * 128
        ntiles = sum(1 for a in range(npad // 128) for b in range(npad // 64) if 64 * b + 63 >= 128 * a)
        kpad = ((T * r + 31) // 32) * 32
        ops = 2.0 * ntiles * 128 * 64 * kpad * (S * (S + 1) // 2)
        ach = ops / (med[2] * 1e-3) / 1e12
        i8_peak = 4500.0
        roof = {"kernel": "gram (k_gram_i8, tcgen05 kind::i8)", "bound": "tensor", "achieved": ach, "peak": i8_peak,
                "unit": "TFLOP/s", "frac": ach / i8_peak,
                "peak_source": "fallback: B200_PROFILING.md nominal dense fp8/int8 4.5 PFLOP/s (MEASURED_PEAKS.json "
                               "has no int8 figure; 2 x its bf16 burst = %.0f)" % (2 * json.load(open(
                                   os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("bf16_tflops", 0.0)
                                   if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 0.0),
                "alg_int8_ops": ops, "digit_slices": S,
                "fp64_equivalent": {"alg_flops": alg["s3_flops_survey"], "achieved": stage_info["gram"]["tflops"],
                                    "peak": fp64, "frac": stage_info["gram"]["tflops"] / fp64, "unit": "TFLOP/s",
                                    "peak_source": "measured in-run (DFMA microbenchmark, rsm_fp64_peak_tflops)"}}
    elif dom in ("gram", "svd"):
        ach = stage_info[dom]["tflops"]
        roof = {"kernel": dom, "bound": "fp64", "achieved": ach, "peak": fp64, "unit": "TFLOP/s",
                "frac": ach / fp64, "peak_source": "measured in-run (DFMA microbenchmark, rsm_fp64_peak_tflops)"}
    else:
        key = {"select": 0, "solve_u": 5, "solve_v": 4}[dom]
        ab = {"select": alg["s1_bytes"], "solve_u": alg["s5_bytes"], "solve_v": alg["s4_bytes"]}[dom]
        ach = ab / (med[key] * 1e-3) / 1e9
        roof = {"kernel": dom, "bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                "peak_source": f"{hbm_src} (MEASURED_PEAKS.json hbm_gbs)"}
    tr = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            tr = json.load(open(tpath)).get(dom)
        except Exception:
            tr = None
    roof["traffic"] = tr

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and Y is not None:
        G = None
        try:
            # the accumulator the reference's solve_v would see (from the device harvest)
            G = ctx.harvest_gram(rsm.TrialParams(rsm.Mode.M2, c["k"], 0, r, r + 1, c["seed"]), T).gram
        except Exception:
            pass
        try:
            cpu = cpu_reference_sample(Y, W, c, G=G, V=F.v)
            cpu["config1_measured"] = cpu_reference_config1()
        except Exception as ex:  # report, never fail the GPU line
            cpu = {"value": None, "unit": "submatrices/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"failed: {ex}"}
    c1 = None
    if rank == 0 and world == 1 and args.config == "config3" and not args.no_cpu_baseline:
        # config 1 on this GPU (device time of one decompose, median of 9), the
        # GPU side of the fully measured config-1 reference comparison
        cc = CONFIGS["config1"]
        ctx1 = rsm.Context(local)
        ctx1.generate(cc["m"], cc["n"], cc["r"], cc["rho"], cc["sigma"], cc["seed"])
        cfg1 = rsm.RsmConfig(rank=cc["r"], mode=rsm.Mode.M2, block=cc["k"], plan=rsm.TrialPlan(cc["T"]),
                             seed=cc["seed"])
        s1 = torch.cuda.ExternalStream(ctx1.stream)
        t1 = []
        for i in range(12):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s1)
            ctx1.decompose(cfg1, fetch=False)
            e1.record(s1)
            e1.synchronize()
            if i >= 3:
                t1.append(e0.elapsed_time(e1))
        ms1 = statistics.median(t1)
        c1 = {"workload": cc["workload"], "ms_per_decompose": ms1, "value": cc["T"] / (ms1 / 1e3),
              "unit": "submatrices/s", "note": "device time, inputs resident (device generator)"}
        ctx1.close()
    stage_info["solve_v"]["solver"] = ctx.solver_stats()
    if args.stages and rank == 0:
        print(json.dumps(stage_info), file=sys.stderr)
    if rank == 0:
        line = {"metric": "submatrices/s (full RSM decompose)", "value": value, "unit": "submatrices/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (reference generator streams, seed 0)",
                "config": arm_config(c, world),
                "e2e": ({"value": T / (e2e_ms / 1e3), "unit": "submatrices/s", "ms_per_step": e2e_ms,
                         "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h} if host_ok else
                        {"value": None, "unit": "submatrices/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
                         "skipped": f"pinned host copy per rank ({host_bytes / 2**30:.0f} GiB x {world}) exceeds "
                                    "HOST_PIN_BUDGET"}),
                "roofline": roof, "stages": stage_info, "cpu_baseline": cpu, "clocks": clk,
                "gpu_launches": launches, "config1": c1,
                "harvest": {"value": T / (float(np.sum(med[:4])) * 1e-3), "unit": "submatrices/s",
                            "note": "T / device time of stages 1-3 (selection, SVD, Gram), SURVEY.md 8(d)"},
                "report": {"e": rep.e, "attempted": rep.trials_attempted, "accepted": rep.trials_accepted,
                           "z": rep.z, "gram_rank": rep.gram_rank, "underdetermined_rows": rep.underdetermined_rows}}
        print(json.dumps(line))
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    ctx.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
