"""Benchmark: HMM forward log-likelihood throughput (observations/s) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NAME] [--impl ours|reference]

One "step" is one full likelihood evaluation (BASELINE.json metric "HMM
observations/sec (log-lik evals/sec)") of the named workload (default
``k25_n1e6``: K=25, N=10^6, BASELINE.json configs[1]) on synthetic
tremor-like data generated with the reference bench recipe
(paper_2003_03508_b200/synth.py).  With N>1 ranks (torchrun) the chain is
N x 10^6 records long and sharded contiguously, 10^6 per GPU ("weak"),
combined with one NCCL all-gather per evaluation.

``value``      obs/s with the stream resident in HBM (the MCMC steady state):
               parameter upload, chain kernel, segment fold, all-gather and
               the 8-byte result download are all inside the timed region.
``e2e``        the same metric through the public array API
               (``_parallel_loglik_arrays`` with pinned host arrays): the
               17 B/record host->device copy is inside the timed region.
``roofline``   chain kernel (the dominant launch), algorithmic 2 K^3 flop per
               record per proposal (reference engine.py:287, 341) / its
               CUDA-event duration, against the measured FP64 DMMA peak.
``cpu_baseline`` the reference package's own engine (baseline/_ref) on all
               host cores, rank 0 at N=1 only, bounded sample.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

# The reference CPU engine runs one numba worker per physical core, each
# calling OpenBLAS dgemm: single-threaded BLAS avoids oversubscription
# (BASELINE.md §2).  Must precede the first numpy import.
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

METRIC = "HMM observations/sec (log-lik evals/sec) at K=25/50/80, 1–8 B200 vs CPU"
UNIT = "obs/s"
# Measured FP64 tensor-core (DMMA m8n8k4) peak on this pool's B200 at 1965 MHz:
# profiles/r1_fp64_peak_microbench.txt (MEASURED_PEAKS.json has no FP64 entry).
FP64_DMMA_PEAK_TFLOPS = 37.1
# Precision-study modes (--precision): dense TF32 tcgen05 peak = half the
# measured dense bf16 peak (MEASURED_PEAKS.json, driver-written; fallback the
# value recorded this round), FP32 SIMT FFMA peak = 148 SMs x 128 lanes x 2 x 1.965 GHz.
FP32_SIMT_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12


def tf32_peak_tflops():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["bf16_tflops"]) / 2.0, "MEASURED_PEAKS.json bf16_tflops / 2"
    except (OSError, KeyError, ValueError):
        return 1629.7 / 2.0, "bf16 1629.7 TF/s (MEASURED_PEAKS.json, round 1) / 2"
L2_FLUSH_BYTES = 256 << 20


def log(msg):
    print(msg, file=sys.stderr, flush=True)


# ---------------------------------------------------------------------------
# clocks
# ---------------------------------------------------------------------------

class ClockSampler:
    FIELDS = ("clocks.sm", "clocks.max.sm", "power.draw", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={','.join(self.FIELDS)}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) != len(self.FIELDS):
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[3:]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU baselines (reference package if installed, else the C oracle port)
# ---------------------------------------------------------------------------

def physical_cores():
    pairs, phys = set(), None
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("physical id"):
                    phys = line.split(":")[1].strip()
                elif line.startswith("core id"):
                    pairs.add((phys, line.split(":")[1].strip()))
    except OSError:
        pass
    return len(pairs) or (os.cpu_count() or 1)


def _reference_module():
    path = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(os.path.join(path, "tremorhmm")):
        sys.path.insert(0, path)
        try:
            import tremorhmm  # noqa: F401
            from tremorhmm import core, engine
            return core, engine
        except Exception as exc:  # pragma: no cover
            log(f"reference package not importable: {exc}")
    return None


def cpu_rate(plist, present, lon, lat, budget_s=12.0, max_reps=5, warmup=0, exact_steps=None):
    """obs/s of the CPU reference on a bounded prefix sample: best of up to
    ``max_reps`` within ``budget_s`` (the cpu_baseline leg), or, with
    ``exact_steps``, ``warmup`` untimed then exactly ``exact_steps`` timed
    evaluations, mean time (the --impl reference arm)."""
    cores = physical_cores()
    threads = cores  # C = physical cores (test_acceptance.py:70-85 counting)
    refmod = _reference_module()
    n = present.size
    k = plist[0].K
    # bounded sample: prefix sized for ~1-3 s per evaluation
    per_obs = 2.0 * k ** 3 / 3e9 / max(threads, 1) + 1.5e-6
    sample = int(min(n, max(20_000, 2.0 / per_obs)))
    pr, lo, la = present[:sample], lon[:sample], lat[:sample]
    params = plist[0]
    if refmod is not None:
        core, engine = refmod
        from tremorhmm import HmmParams, StateEmission
        rp = HmmParams(gamma=params.gamma, delta=params.delta,
                       states=tuple(StateEmission(s.p, s.mu, s.sigma) for s in params.states))
        cfg = engine.EngineConfig(workers=threads, segments=threads)
        engine._parallel_loglik_arrays(rp, pr[:64], lo[:64], la[:64], cfg)  # numba warm-up (bench.py:66-68)
        fn = lambda: engine._parallel_loglik_arrays(rp, pr, lo, la, cfg)  # noqa: E731
        kind = "reference"
        desc = f"tremorhmm engine._parallel_loglik_arrays(workers={threads}, segments={threads})"
        ser_fn = lambda m: core._forward_loglik_arrays(rp, pr[:m], lo[:m], la[:m], 1)  # noqa: E731
    else:
        from oracle import coracle
        fn = lambda: coracle.parallel_loglik(params, pr, lo, la, threads, threads=threads)  # noqa: E731
        kind = "port"
        desc = f"oracle/thmm_oracle.c segmented engine, {threads} threads"
        ser_fn = lambda m: coracle.forward_loglik(params, pr[:m], lo[:m], la[:m], 1)  # noqa: E731
    times = []
    if exact_steps is not None:
        for _ in range(warmup):
            fn()
        for _ in range(exact_steps):
            t0 = time.perf_counter()
            fn()
            times.append(time.perf_counter() - t0)
        best = statistics.mean(times)
    else:
        t_start = time.perf_counter()
        while len(times) < max_reps and (time.perf_counter() - t_start) < budget_s:
            t0 = time.perf_counter()
            fn()
            times.append(time.perf_counter() - t0)
        best = min(times)
    # serial Algorithm 1 on one core, 2e4-record prefix
    m = min(sample, 20_000)
    t0 = time.perf_counter()
    ser_fn(m)
    ser = m / (time.perf_counter() - t0)
    return dict(value=sample / best, unit=UNIT,
                cores=threads, kind=kind, logical_cpus=os.cpu_count(),
                sample=f"{desc}; prefix of {sample} records of the workload chain, "
                       + (f"mean of {len(times)} timed after {warmup} warm-up" if exact_steps is not None
                          else f"best of {len(times)}"),
                serial_1core_obs_per_s=ser, physical_cores=cores, reps=len(times), seconds_per_eval=best)


# ---------------------------------------------------------------------------
# main
# ---------------------------------------------------------------------------

def runs_steps(present, nseg, R, W=32):
    """Steps of the run-absorbing chain (csrc/thmm_runs.cuh) over `present`
    cut into nseg reference segments: a record starts a step when present, or
    absent at a run position (from the last present record or the start of its
    32-record window of the segment) that is a multiple of R."""
    n = present.size
    s = np.arange(nseg, dtype=np.int64)
    seg_lo = s * (n // nseg) + np.minimum(s, n % nseg)  # reference segment_bounds (engine.py:97-111)
    seg_len = np.diff(np.append(seg_lo, n))
    idx = np.arange(n, dtype=np.int64)
    pos = idx - np.repeat(seg_lo, seg_len)
    lp = np.maximum.accumulate(np.where(present, idx, -1))
    rstart = np.maximum(np.concatenate([[-1], lp[:-1]]) + 1, idx - pos % W)
    return int(np.count_nonzero(present | ((idx - rstart) % R == 0)))


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=600)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="k25_n1e6")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--e2e-steps", type=int, default=100,
                    help="upper bound; the e2e leg runs at most ~3 s (at least 3 steps)")
    ap.add_argument("--dist-mode", default="auto", choices=["auto", "chain", "proposals"],
                    help="under torchrun: shard the chain (chain) or the batched proposals (proposals); "
                         "auto = chain for single-proposal workloads, proposals for batches")
    ap.add_argument("--precision", default="float64", choices=["float64", "float32", "tf32", "tf32x2", "tf32x3"],
                    help="float64 = the parity path (headline); the others are the precision study")
    return ap.parse_args()


def dist_init(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # Under torchrun (WORLD_SIZE set, even =1) the sharded NCCL path is used.
    use_dist = "WORLD_SIZE" in os.environ
    if use_dist:
        import torch
        import torch.distributed as dist
        # Test hook: THMM_BENCH_BACKEND=gloo with THMM_BENCH_ONE_GPU=1 runs every rank
        # on cuda:0 (exercises the multi-rank path on a single-GPU box).
        if os.environ.get("THMM_BENCH_ONE_GPU") == "1":
            local = 0
        torch.cuda.set_device(local)
        backend = os.environ.get("THMM_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return world, rank, local, use_dist


def make_data(args, world):
    from paper_2003_03508_b200 import synth

    w = synth.WORKLOADS[args.workload]
    n = w["n"] * world if w["batch"] == 1 else w["n"]
    plist, pr, lo, la = synth.make_workload(args.workload, n=n)
    return w, plist, pr, lo, la


def run_reference(args):
    world, rank, _ = int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), 0
    if rank != 0:
        return
    from paper_2003_03508_b200 import synth

    w = synth.WORKLOADS[args.workload]
    plist, pr, lo, la = synth.make_workload(args.workload)
    res = cpu_rate(plist[:1], pr, lo, la, warmup=args.warmup, exact_steps=args.steps)
    value = res["value"]
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": res["reps"], "warmup": args.warmup, "ms_per_step": res["seconds_per_eval"] * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference bench recipe: prior draw + simulate_path, seeded)",
        "config": {"workload": args.workload, "K": w["k"], "N": w["n"] * (world if w["batch"] == 1 else 1),
                   "batch": w["batch"], "parallelism": "cpu threads (rank 0 only); rate measured on the "
                   "first proposal over a prefix sample of the chain"},
        "cpu_baseline": {k: res[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "serial_1core_obs_per_s": res["serial_1core_obs_per_s"],
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    assert args.warmup >= 3, "at least 3 warm-up steps"
    import torch

    world, rank, local, use_dist = dist_init(args)
    torch.cuda.set_device(local)
    import paper_2003_03508_b200 as eng
    from paper_2003_03508_b200 import _native

    _native.require_device()
    eng.set_default_device(local)
    w, plist, pr, lo, la = make_data(args, world)
    n_total = pr.size
    B = len(plist)
    K = plist[0].K
    cfg = eng.EngineConfig(precision=args.precision)
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream

    mode = args.dist_mode if args.dist_mode != "auto" else ("chain" if B == 1 else "proposals")
    b_local = B
    if use_dist and mode == "proposals":
        import torch.distributed as dist
        from paper_2003_03508_b200.distributed import ReplicaLoglik

        # every rank holds the whole chain and evaluates its slice of the proposals
        replica = ReplicaLoglik(pr, lo, la, device=local)
        n_local = n_total
        b_lo, b_hi = eng.segment_bounds(B, world)[rank] if B >= world else (min(rank, B), min(rank + 1, B))
        b_local = b_hi - b_lo
        call = lambda: replica.loglik_batch(plist, cfg, stream=sptr)  # noqa: E731
        barrier = dist.barrier
    elif use_dist:
        import torch.distributed as dist
        from paper_2003_03508_b200.distributed import ShardedLoglik

        sharded = ShardedLoglik(pr, lo, la, device=local)
        n_local = sharded.n_local
        call = lambda: sharded.loglik_batch(plist, cfg, stream=sptr)  # noqa: E731
        barrier = dist.barrier
    else:
        dev = eng.DeviceObservations(pr, lo, la, device=local)
        n_local = n_total
        call = lambda: dev.loglik_batch(plist, cfg, stream=sptr)  # noqa: E731
        barrier = lambda: None  # noqa: E731

    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")
    _native.profile_enable(True)
    for _ in range(args.warmup):
        vals = call()
    torch.cuda.synchronize()

    sampler = ClockSampler(local)
    sampler.start()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    chain_ms, fold_ms, launches = [], [], 0
    barrier()
    torch.cuda.synchronize()
    for i in range(args.steps):
        flush.zero_()  # L2 flush outside the timed interval of each step
        ev[i][0].record(stream)
        vals = call()
        ev[i][1].record(stream)
        if use_dist and mode == "chain":
            c, f, nseg = sharded.last_profile
            launches += sharded.last_launches
        else:
            c, f, nseg = _native.profile_last()
            launches += _native.last_launch_count()
        chain_ms.append(c)
        fold_ms.append(f)
    torch.cuda.synchronize()
    barrier()
    clocks = sampler.stop()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = sum(step_ms)
    red_dev = "cuda" if (not use_dist or dist.get_backend() == "nccl") else "cpu"
    if use_dist:
        t = torch.tensor([total_ms], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = B * n_total / (ms_per_step / 1e3)

    # ---- roofline of the chain kernel (dominant launch) -----------------
    runs = _native.profile_runs()  # the timed calls ran the run-absorbing chain
    plan = _native.plan_info(K, args.precision, local)
    chain_avg = statistics.mean(chain_ms)
    flops = 2.0 * K ** 3 * n_local * b_local
    extra = {}
    if runs:
        # Algorithmic work of the run-absorbing chain: one K x K product (2K^3
        # flop) per STEP -- a present record or a chunk of up to R absent
        # records -- counted exactly with the kernel's rule on this rank's records.
        kp = eng.padded_states(K)
        nt, skip = kp // 8, K % 8 == 1
        obs_handle = dev if not use_dist else (sharded.obs if mode == "chain" else replica.obs)
        rinfo = obs_handle.runs_info(K, args.precision)
        R = rinfo["R"]
        if use_dist and mode == "chain":
            lo_r, hi_r = eng.segment_bounds(n_total, world)[rank]
        else:
            lo_r, hi_r = 0, n_total
        steps = runs_steps(pr[lo_r:hi_r], nseg, R)
        plan = {"nt": K // 8 if (K >= 9 and 1 <= K % 8 <= 4) else nt, "tail": K % 8 if (K >= 9 and 1 <= K % 8 <= 4) else 0,
                "G": rinfo["G"], "W": rinfo["W"], "regs": rinfo["regs"], "ctas_per_sm": rinfo["ctas_per_sm"]}
        flops = 2.0 * K ** 3 * steps * b_local
        nh = K // 8 if (K >= 9 and 1 <= K % 8 <= 4) else nt  # DMMA head tiles (K % 8 in 1..4: SIMT tail)
        dmma = nt * (2 * nh * nh - (nh if (skip and nh == nt) else 0))  # DMMA.8x8x4 per segment-step
        extra = {"algorithm": "run-absorbing chain: absent runs applied as precomputed (Gamma Q)^r, r <= R",
                 "R": R, "steps": steps * b_local, "steps_per_record": steps / max(hi_r - lo_r, 1),
                 "executed_dmma_tflops": dmma * 512.0 * steps * b_local / (chain_avg / 1e3) / 1e12,
                 "reference_equivalent_tflops": 2.0 * K ** 3 * n_local * b_local / (chain_avg / 1e3) / 1e12,
                 "note": "achieved = 2K^3 per step / chain time; reference_equivalent counts 2K^3 per record "
                         "(the record-by-record algorithm's work) over the same time"}
    achieved = flops / (chain_avg / 1e3) / 1e12
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "r1_traffic.json")
    if os.path.exists(tpath):
        for t in json.load(open(tpath)).get("entries", []):
            if (t["workload"] == args.workload and t["precision"] == args.precision
                    and t.get("kernel", "").startswith("chain_runs") == runs):
                traffic = (t["dram_read"] + t["dram_write"]) * n_local / t["n"]
    if runs:
        peak, peak_src = FP64_DMMA_PEAK_TFLOPS, "measured FP64 DMMA m8n8k4 microbenchmark, profiles/r1_fp64_peak_microbench.txt"
        kernel = f"chain_runs_kernel<nt={plan['nt']}, skip={int(skip and plan['tail'] == 0)}, tail={plan['tail']}> (R={R})"
    elif args.precision == "float64":
        peak, peak_src = FP64_DMMA_PEAK_TFLOPS, "measured FP64 DMMA m8n8k4 microbenchmark, profiles/r1_fp64_peak_microbench.txt"
        kernel = "chain_f64_kernel<nt={nt}, skip={skip}, tail={tail}>".format(
            nt=plan["nt"], skip=int(plan["tail"] == 0 and K % 8 == 1), tail=plan["tail"])
    elif args.precision == "float32":
        peak, peak_src = FP32_SIMT_PEAK_TFLOPS, "FP32 FFMA issue peak, 148 SM x 128 lanes x 2 flop x 1.965 GHz"
        kernel = f"chain_f32_kernel<{plan['nt']}>"
    else:
        tf, src = tf32_peak_tflops()
        passes = {"tf32": 1, "tf32x2": 2, "tf32x3": 3}[args.precision]
        peak, peak_src = tf / passes, f"dense TF32 tcgen05 = {src}" + (f" / {passes} ({passes} MMAs per product)"
                                                                        if passes > 1 else "")
        kernel = f"chain_tc_kernel<NP={plan['nt']}, KP={plan['tail']}> ({args.precision}, {plan['W']} warps)"
    roofline = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak, "traffic": traffic,
                "traffic_note": "bytes/launch from the committed ncu capture (profiles/r1_traffic.json), "
                                "scaled to this launch's records; algorithmic 17 B/record",
                "kernel": kernel, "plan": plan, "peak_source": peak_src,
                "flops_per_launch": flops, "chain_ms": chain_avg, "fold_ms": statistics.mean(fold_ms),
                "chain_share_of_step": chain_avg / ms_per_step, "segments": nseg, **extra}

    _native.profile_enable(False)  # the e2e leg is timed on the host clock; no per-call event pairs
    # ---- e2e through the public array API with pinned host buffers -------
    if not use_dist:
        pin_pr = torch.from_numpy(pr.view(np.uint8)).pin_memory().numpy().view(np.bool_)
        pin_lo = torch.from_numpy(lo).pin_memory().numpy()
        pin_la = torch.from_numpy(la).pin_memory().numpy()
        e2e_fn = lambda: (eng.parallel_loglik_batch(plist, (pin_pr, pin_lo, pin_la), cfg)  # noqa: E731
                          if B > 1 else eng._parallel_loglik_arrays(plist[0], pin_pr, pin_lo, pin_la, cfg))
        h2d = n_total * 17
    elif mode == "proposals":
        pin_full = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy() for a in (pr.view(np.uint8), lo, la)]
        e2e_fn = lambda: replica.loglik_batch(plist, cfg, stream=sptr,  # noqa: E731
                                              host=(pin_full[0].view(np.bool_), pin_full[1], pin_full[2]))
        h2d = n_total * 17
    else:
        lo_r, hi_r = eng.segment_bounds(n_total, world)[rank]
        pin = [torch.from_numpy(np.ascontiguousarray(a[lo_r:hi_r])).pin_memory().numpy()
               for a in (pr.view(np.uint8), lo, la)]
        e2e_fn = lambda: sharded_e2e(pin)  # noqa: E731

        def sharded_e2e(pin):
            return sharded.loglik_batch(plist, cfg, stream=sptr, host_shard=(pin[0].view(np.bool_), pin[1], pin[2]))
        h2d = (hi_r - lo_r) * 17
    h2d += B * (K * K + 9 * K) * 8
    # warm-up: >= 3 calls and ~0.3 s of device time (the first ~40 host-array
    # calls after the device-timed leg can run up to 40% slow -- clock-sampler
    # teardown, host graph capture; see tools/e2e_blocks.py).  The count comes
    # from ms_per_step (max-reduced), so every rank runs the same number of
    # collective steps.
    for _ in range(max(3, min(500, int(0.3 / max(ms_per_step / 1e3, 1e-6))))):
        e2e_fn()
    e2e_steps = max(3, min(args.e2e_steps, int(3.0 / max(ms_per_step / 1e3, 1e-6))))
    if use_dist:  # every rank must run the same number of collective steps
        t = torch.tensor([e2e_steps], dtype=torch.int64, device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        e2e_steps = int(t.item())
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    marks = []
    for i in range(e2e_steps):
        e2e_fn()
        if (i + 1) % 20 == 0:
            marks.append(time.perf_counter())
    torch.cuda.synchronize()
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    if marks:
        blocks = np.diff([t0] + marks) / 20 * 1e3
        log("e2e ms/step per 20-call block: " + " ".join(f"{x:.3f}" for x in blocks))
    if use_dist:
        t = torch.tensor([e2e_s], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e = {"value": B * n_total / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "steps": e2e_steps,
           "d2h_bytes_per_step": int(B * 12), "ms_per_step": e2e_s * 1e3,
           "api": "paper_2003_03508_b200._parallel_loglik_arrays (pinned host numpy arrays)",
           "transfer": ("zero-copy: the chain kernels read the pinned arrays in place over PCIe every call "
                        "(uncached ld.global.cv, coordinates of present records only; ncu: 13.3 MB PCIe reads per "
                        "K=25 N=1e6 call, profiles/r1_mapped_pcie_ncu.csv); h2d_bytes_per_step counts the input "
                        "arrays" + ("" if not use_dist else "; under torchrun each rank reads its own pinned shard"))}

    # ---- parity of the timed result vs the golden -------------------------
    parity = None
    gold_path = os.path.join(ROOT, "tests", "golden", "bench_configs.json")
    if world == 1 and os.path.exists(gold_path):
        g = json.load(open(gold_path))["workloads"].get(args.workload)
        if g is not None:
            want = np.array(g["loglik"])
            parity = float(np.max(np.abs(np.asarray(vals) - want) / np.abs(want)))

    # Host-side proposal cost for batched workloads (reported
    # separately): B parameter vectors -> packed C-ABI block, vectorised.
    host_prop = None
    if B > 1:
        from paper_2003_03508_b200 import proposals

        vecs = proposals.params_to_vectors(plist)
        proposals.params_from_vectors(K, vecs, "uniform")
        t0 = time.perf_counter()
        for _ in range(5):
            proposals.params_from_vectors(K, vecs, "uniform")
        host_prop = {"ms_per_batch": (time.perf_counter() - t0) / 5 * 1e3, "batch": B,
                     "what": "proposals.params_from_vectors (vector -> validated packed block), delta uniform"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            cpu = cpu_rate(plist[:1], pr, lo, la)
        except Exception as exc:  # pragma: no cover
            cpu = {"error": repr(exc)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            # single-proposal workloads grow the chain with the GPU count (10^6 records per GPU);
            # the 256-proposal batch keeps its 10^6-record chain and shards it ("strong")
            "scaling": "weak" if w["batch"] == 1 else "strong", "vs_baseline": None,
            "dtype": {"float64": "f64", "float32": "f32"}.get(args.precision, args.precision),
            "data": "synthetic (reference bench recipe: prior draw + simulate_path, seeded; "
                    "paper_2003_03508_b200/synth.py)",
            "config": {"workload": args.workload, "K": K, "N": n_total, "N_per_gpu": n_local, "batch": B,
                       "segments_per_gpu": nseg,
                       "parallelism": ("1 GPU" if not use_dist else
                                       (f"chain-sharded x{world} (range nodes exchanged by peer-memory stores over "
                                        f"NVLink + epoch flags)" if getattr(sharded, "transport_used", None) == "peer"
                                        else f"chain-sharded x{world} (NCCL all-gather of range nodes)")
                                       if mode == "chain"
                                       else f"proposal-sharded x{world} (NCCL all-gather of B logL values)"),
                       "l2": "flushed (256 MiB write) before every timed step"},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks,
            "gpu_launches": launches, "parity_max_rel_vs_reference": parity,
            **({"host_proposal_pack": host_prop} if host_prop else {}),
        }
        print(json.dumps(line), flush=True)
    if use_dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
