"""Benchmark: HMM forward log-likelihood throughput (observations/s) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NAME] [--impl ours|reference]

One "step" is one full likelihood evaluation (BASELINE.json metric "HMM
observations/sec (log-lik evals/sec)") of the named workload on synthetic
tremor-like data generated with the reference bench recipe
(paper_2003_03508_b200/synth.py).  Default workload ``k80_n1e8``: K=80,
N=10^8 (BASELINE.json configs[3], the north-star target and the largest
configuration that fits one GPU), FP64.  The K=25 N=10^6 (configs[1]), K=50
N=10^7 (configs[2]) and 256-proposal (configs[4]) workloads are measured in
the same run and reported as ``subconfigs`` of the same line.

Under torchrun (N>1 ranks) the chain keeps its length ("strong" scaling,
BASELINE configs[2]/[3]: fixed N across 2/4/8 GPUs): rank r holds records
``segment_bounds(N, world)[r]`` only.  Stitched combine (default when every
shard is long enough): each rank reduces its shard to its final forward row
and log-scale, ONE NCCL all-gather, each rank links the previous rank's row
into its first segment, ONE more all-gather of 2 doubles per proposal, a
rank-order sum; otherwise one scaled K x K node per rank is all-gathered and
folded in rank order (``THMM_TRANSPORT=nccl``, the default; ``peer`` selects
the NVLink peer-memory mailbox).  The 256-proposal batch shards proposals.

``value``      obs/s with the stream resident in HBM (the MCMC steady state):
               parameter upload, chain kernels, combine, all-gathers and
               the 8-byte result download are all inside the timed region.
``e2e``        the same metric through the public array API
               (``_parallel_loglik_arrays``) from PAGEABLE host numpy arrays
               -- what the reference's MCMC driver passes on every call
               (bayes.py:712-715): the 17 B/record host->device transfer is
               inside the timed region (the arrays are page-locked in place on
               the first call, ``first_call_ms``; then staged by DMA in time
               chunks under the chain, or read over PCIe in place for sparse
               streams).  ``e2e.pinned`` is the same from pinned arrays,
               ``e2e.batch_b256`` the 256-proposal batch (configs[4]).
``roofline``   the dominant kernel of the path that ran (the stitched main
               pass: 2 K^2 flop per record -- one row times Gamma; matrix
               paths: 2 K^3 per K x K product, reference engine.py:287, 341)
               / its CUDA-event duration, against the measured FP64 DMMA peak;
               ``ncu_pipe_active`` from the committed ncu capture.
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
    """obs/s of the CPU reference on the chain or a bounded prefix sample: mean
    of up to ``max_reps`` within ``budget_s`` (the cpu_baseline leg), or, with
    ``exact_steps``, ``warmup`` untimed then exactly ``exact_steps`` timed
    evaluations, mean time (the --impl reference arm)."""
    cores = physical_cores()
    threads = cores  # C = physical cores (test_acceptance.py:70-85 counting)
    refmod = _reference_module()
    n = present.size
    k = plist[0].K
    # the whole chain when one evaluation costs <= ~1 s, else a bounded prefix
    # sample sized for ~2 s per evaluation (the rate is per record: the
    # reference's serial forward is linear in N, test_output.txt:16); the
    # per-record cost is calibrated on a 50k-record prefix
    params = plist[0]
    if refmod is not None:
        core, engine = refmod
        from tremorhmm import HmmParams, StateEmission
        rp = HmmParams(gamma=params.gamma, delta=params.delta,
                       states=tuple(StateEmission(s.p, s.mu, s.sigma) for s in params.states))
        cfg = engine.EngineConfig(workers=threads, segments=threads)
        engine._parallel_loglik_arrays(rp, present[:64], lon[:64], lat[:64], cfg)  # numba warm-up (bench.py:66-68)
        m0 = min(n, 50_000)
        t0 = time.perf_counter()
        engine._parallel_loglik_arrays(rp, present[:m0], lon[:m0], lat[:m0], cfg)
        per_obs = (time.perf_counter() - t0) / m0
        sample = n if n * per_obs <= 1.0 else int(min(n, max(m0, 2.0 / per_obs)))
        pr, lo, la = present[:sample], lon[:sample], lat[:sample]
        fn = lambda: engine._parallel_loglik_arrays(rp, pr, lo, la, cfg)  # noqa: E731
        kind = "reference"
        desc = f"tremorhmm engine._parallel_loglik_arrays(workers={threads}, segments={threads})"
        ser_fn = lambda m: core._forward_loglik_arrays(rp, pr[:m], lo[:m], la[:m], 1)  # noqa: E731
    else:
        from oracle import coracle
        per_obs = 2.0 * k ** 3 / 3e9 / max(threads, 1) + 1.5e-6
        sample = n if n * per_obs <= 1.0 else int(min(n, max(20_000, 2.0 / per_obs)))
        pr, lo, la = present[:sample], lon[:sample], lat[:sample]
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
        best = statistics.mean(times)  # same statistic as the --impl reference arm
    # serial Algorithm 1 on one core, 2e4-record prefix
    m = min(sample, 20_000)
    t0 = time.perf_counter()
    ser_fn(m)
    ser = m / (time.perf_counter() - t0)
    return dict(value=sample / best, unit=UNIT, sample_records=sample,
                cores=threads, kind=kind, logical_cpus=os.cpu_count(),
                sample=f"{desc}; " + ("the whole chain" if sample == n else
                                       f"prefix of {sample} of the workload's {n} records") + ", "
                       + (f"mean of {len(times)} timed after {warmup} warm-up" if exact_steps is not None
                          else f"mean of {len(times)}"),
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


def runs_steps_chunked(present, nseg, R, W=32, chunk=8_000_000):
    """runs_steps over whole segments at a time (bounded host memory at N=10^8)."""
    n = present.size
    bounds = [(s * (n // nseg) + min(s, n % nseg)) for s in range(nseg + 1)]
    total, s0 = 0, 0
    while s0 < nseg:
        s1 = s0 + 1
        while s1 < nseg and bounds[s1 + 1] - bounds[s0] <= chunk:
            s1 += 1
        part = present[bounds[s0]:bounds[s1]]
        # the sub-range is cut into s1 - s0 segments exactly as the full split does
        total += runs_steps(part, s1 - s0, R, W)
        s0 = s1
    return total


SUBCONFIGS = ("k25_n1e6", "k50_n1e7", "k25_n1e6_b256")
L2_NOTE = "flushed (256 MiB write) before every timed step"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="k80_n1e8")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--e2e-steps", type=int, default=100,
                    help="upper bound; each e2e leg runs at most ~3 s (at least 3 steps)")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="under torchrun: strong = the workload's N across all GPUs (BASELINE configs[2]/[3]); "
                         "weak = N records per GPU")
    ap.add_argument("--dist-mode", default="auto", choices=["auto", "chain", "proposals"],
                    help="under torchrun: shard the chain (chain) or the batched proposals (proposals); "
                         "auto = chain for single-proposal workloads, proposals for batches")
    ap.add_argument("--precision", default="float64", choices=["float64", "float32", "tf32", "tf32x2", "tf32x3"],
                    help="float64 = the parity path (headline); the others are the precision study")
    ap.add_argument("--subconfigs", default=",".join(SUBCONFIGS),
                    help="comma-separated workloads also measured and reported under 'subconfigs' ('none': skip)")
    ap.add_argument("--sub-steps", type=int, default=20)
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
            # communicator init lines (ranks, devices, NVLink/NVLS topology) in the log
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return world, rank, local, use_dist


def workload_n(name, world, scaling):
    from paper_2003_03508_b200 import synth

    w = synth.WORKLOADS[name]
    return w["n"] * world if (scaling == "weak" and w["batch"] == 1) else w["n"]


def config_dict(name, world, scaling):
    """The workload's config -- identical in this arm and the --impl reference arm."""
    from paper_2003_03508_b200 import synth

    w = synth.WORKLOADS[name]
    return {"workload": name, "K": w["k"], "N": workload_n(name, world, scaling), "batch": w["batch"],
            "seed": w["seed"], "l2": L2_NOTE}


def golden_loglik(name, n):
    gold_path = os.path.join(ROOT, "tests", "golden", "bench_configs.json")
    if not os.path.exists(gold_path):
        return None
    g = json.load(open(gold_path))["workloads"].get(name)
    if g is None or int(g["n"]) != int(n):
        return None
    return np.array(g["loglik"])


def run_reference(args):
    world, rank = int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2003_03508_b200 import synth

    w = synth.WORKLOADS[args.workload]
    n = workload_n(args.workload, world, args.scaling)
    plist, pr, lo, la = synth.make_workload(args.workload, n=n)
    res = cpu_rate(plist[:1], pr, lo, la, warmup=args.warmup, exact_steps=args.steps)
    value = res["value"]
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": res["reps"], "warmup": args.warmup, "ms_per_step": res["seconds_per_eval"] * 1e3,
        "higher_is_better": True, "scaling": args.scaling if w["batch"] == 1 else "strong", "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (reference bench recipe: prior draw + simulate_path, seeded)",
        "config": config_dict(args.workload, world, args.scaling),
        "run": {"parallelism": f"CPU, {res['cores']} threads on rank 0 (reference engine, "
                               "workers = segments = physical cores)",
                "sample_records": res["sample_records"],
                "rate": "obs/s of the first proposal over the sample (the engine is linear in N)"},
        "cpu_baseline": {k: res[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "serial_1core_obs_per_s": res["serial_1core_obs_per_s"],
    }
    print(json.dumps(line), flush=True)


class Ctx:
    """Process-group context of one bench run."""

    def __init__(self, world, rank, local, use_dist):
        self.world, self.rank, self.local, self.use_dist = world, rank, local, use_dist
        if use_dist:
            import torch.distributed as dist

            self.dist = dist
            self.red_dev = "cuda" if dist.get_backend() == "nccl" else "cpu"

    def barrier(self):
        if self.use_dist:
            self.dist.barrier()

    def reduce(self, x, op="max", dtype=None):
        if not self.use_dist:
            return x
        import torch

        t = torch.tensor([x], dtype=dtype or torch.float64, device=self.red_dev)
        self.dist.all_reduce(t, op={"max": self.dist.ReduceOp.MAX, "min": self.dist.ReduceOp.MIN}[op])
        return t.item()

    def gather(self, obj):
        if not self.use_dist:
            return [obj]
        out = [None] * self.world
        self.dist.all_gather_object(out, obj)
        return out


def time_host_leg(ctx, fn, ms_hint, max_steps, label):
    """Host-clock timing of an end-to-end leg (every rank runs the same number
    of calls; max over ranks).  Warm-up: >= 2 calls and ~0.3 s (the first
    host-array calls after the device-timed leg run slow on some boxes:
    clock-sampler teardown, host graph capture)."""
    import torch

    torch.cuda.synchronize()
    t0 = time.perf_counter()
    fn()
    torch.cuda.synchronize()
    first = time.perf_counter() - t0
    for _ in range(max(1, min(500, int(0.3 / max(ms_hint / 1e3, 1e-6))))):
        fn()
    steps = max(3, min(max_steps, int(3.0 / max(ms_hint / 1e3, 1e-6))))
    steps = int(ctx.reduce(steps, "min", torch.int64))
    ctx.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    marks = []
    for i in range(steps):
        fn()
        if (i + 1) % 20 == 0:
            marks.append(time.perf_counter())
    torch.cuda.synchronize()
    sec = (time.perf_counter() - t0) / steps
    if marks:
        blocks = np.diff([t0] + marks) / 20 * 1e3
        log(f"{label}: e2e ms/step per 20-call block: " + " ".join(f"{x:.3f}" for x in blocks))
    return ctx.reduce(sec, "max"), steps, ctx.reduce(first, "max")


def measure(ctx, args, name, steps, warmup, main):
    """Device-resident throughput, roofline, parity and the end-to-end legs of
    one workload; returns the per-workload part of the JSON line."""
    import torch

    import paper_2003_03508_b200 as eng
    from paper_2003_03508_b200 import _native, synth

    world, rank, local, use_dist = ctx.world, ctx.rank, ctx.local, ctx.use_dist
    w = synth.WORKLOADS[name]
    n_total = workload_n(name, world, args.scaling)
    t_syn = time.perf_counter()
    plist, pr, lo, la = synth.make_workload(name, n=n_total)
    t_syn = time.perf_counter() - t_syn
    B, K = len(plist), plist[0].K
    cfg = eng.EngineConfig(precision=args.precision)
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream
    mode = args.dist_mode if args.dist_mode != "auto" else ("chain" if B == 1 else "proposals")
    transport = os.environ.get("THMM_TRANSPORT", "nccl")
    b_local, lo_r, hi_r = B, 0, n_total
    sharded = replica = dev = None
    if use_dist and mode == "proposals":
        from paper_2003_03508_b200.distributed import ReplicaLoglik

        # every rank holds the whole chain and evaluates its slice of the proposals
        replica = ReplicaLoglik(pr, lo, la, device=local)
        b_lo, b_hi = eng.segment_bounds(B, world)[rank] if B >= world else (min(rank, B), min(rank + 1, B))
        b_local = b_hi - b_lo
        call = lambda: replica.loglik_batch(plist, cfg, stream=sptr)  # noqa: E731
        obs_handle = replica.obs
    elif use_dist:
        from paper_2003_03508_b200.distributed import ShardedLoglik

        sharded = ShardedLoglik(pr, lo, la, device=local, transport=transport)
        lo_r, hi_r = eng.segment_bounds(n_total, world)[rank]
        call = lambda: sharded.loglik_batch(plist, cfg, stream=sptr)  # noqa: E731
        obs_handle = sharded.obs
    else:
        dev = eng.DeviceObservations(pr, lo, la, device=local)
        call = lambda: dev.loglik_batch(plist, cfg, stream=sptr)  # noqa: E731
        obs_handle = dev
    n_local = hi_r - lo_r

    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")
    _native.profile_enable(True)
    for _ in range(warmup):
        vals = call()
    torch.cuda.synchronize()

    sampler = ClockSampler(local)
    sampler.start()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    chain_ms, fold_ms, phases, launches = [], [], [], 0
    ctx.barrier()
    torch.cuda.synchronize()
    for i in range(steps):
        flush.zero_()  # L2 flush outside the timed interval of each step
        ev[i][0].record(stream)
        vals = call()
        ev[i][1].record(stream)
        if sharded is not None:
            c, f, nseg = sharded.last_profile
            launches += sharded.last_launches
        else:
            c, f, nseg = _native.profile_last()
            launches += _native.last_launch_count()
        chain_ms.append(c)
        fold_ms.append(f)
        phases.append(_native.profile_phases())
    torch.cuda.synchronize()
    ctx.barrier()
    clocks = sampler.stop()
    total_ms = ctx.reduce(sum(a.elapsed_time(b) for a, b in ev), "max")
    ms_per_step = total_ms / steps
    value = B * n_total / (ms_per_step / 1e3)
    runs = _native.profile_runs()  # the timed calls ran the run-absorbing chain
    transport_used = getattr(sharded, "transport_used", None) if sharded is not None else None

    # ---- roofline of the chain kernel (dominant launch) -----------------
    plan = _native.plan_info(K, args.precision, local)
    chain_avg = statistics.mean(chain_ms)
    flops = 2.0 * K ** 3 * n_local * b_local
    extra = {}
    pmode = phases[-1][0] if phases else 0
    kp = eng.padded_states(K)
    split = K >= 9 and 1 <= K % 8 <= 4
    nh = K // 8 if split else kp // 8  # DMMA head tiles (K % 8 in 1..4: SIMT tail)
    tile_dmma = 2 * nh * nh - (nh if (K % 8 == 1 and not split) else 0)  # DMMA.8x8x4 per 8-row tile and step
    dom_ms = chain_avg  # duration of the dominant kernel
    if pmode == 2:
        # Stitched chain (csrc/thmm_vec.cuh): ONE forward row per segment,
        # 8 segments per DMMA tile: 2K^2 flop per record per proposal in the
        # main pass (chain_fwd_kernel, the dominant launch); links add ~2 rows x
        # 8-48 records per segment.
        main_ms = max(statistics.mean(p[1] for p in phases), 1e-9)
        link_ms = statistics.mean(p[2] for p in phases)
        dom_ms = main_ms
        flops = 2.0 * K * K * n_local * b_local
        extra = {"algorithm": "stitched chain: one forward row per segment (8 segments per DMMA tile), "
                              "consecutive segments linked once two rows are proportional (2^-40)",
                 "main_pass_ms": main_ms, "link_ms": link_ms,
                 "executed_dmma_tflops": tile_dmma * 512.0 * n_local * b_local / 8 / (main_ms / 1e3) / 1e12,
                 "reference_equivalent_tflops": 2.0 * K ** 3 * n_local * b_local / (chain_avg / 1e3) / 1e12,
                 "note": "achieved = 2K^2 per record (one K-vector x K x K product) / main-pass time; "
                         "reference_equivalent counts the record-by-record algorithm's 2K^3 per record over "
                         "the whole chain phase"}
        kernel = f"chain_fwd_kernel<nt={nh}, skip={int(K % 8 == 1 and not split)}, tail={K % 8 if split else 0}>"
    elif pmode == 1:
        burn_ms = statistics.mean(p[1] for p in phases)
        vec_ms = max(statistics.mean(p[2] for p in phases), 1e-9)
        st = _native.collapse_stats(obs_handle._handle)
        burned = st.get("burn_records", 0.0)
        dom_ms = vec_ms
        flops = 2.0 * K * K * max(n_local * b_local - burned, 0.0)
        extra = {"algorithm": "rank-one collapse: run-absorbing burn-in until each segment product is rank one "
                              "(2^-40), then one row per segment (8 per DMMA tile)",
                 "burn_in_ms": burn_ms, "vector_ms": vec_ms, "burn_in_records": burned,
                 "executed_dmma_tflops": tile_dmma * 512.0 * max(n_local * b_local - burned, 0.0) / 8
                 / (vec_ms / 1e3) / 1e12,
                 "reference_equivalent_tflops": 2.0 * K ** 3 * n_local * b_local / (chain_avg / 1e3) / 1e12}
        kernel = f"chain_vec_kernel<nt={nh}, skip={int(K % 8 == 1 and not split)}, tail={K % 8 if split else 0}>"
    elif runs:
        # Algorithmic work of the run-absorbing chain: one K x K product (2K^3
        # flop) per STEP -- a present record or a chunk of up to R absent
        # records -- counted exactly with the kernel's rule on this rank's records.
        kp = eng.padded_states(K)
        nt, skip = kp // 8, K % 8 == 1
        rinfo = obs_handle.runs_info(K, args.precision)
        R = rinfo["R"]
        nsteps = runs_steps_chunked(pr[lo_r:hi_r], nseg, R)
        plan = {"nt": K // 8 if split else nt, "tail": K % 8 if split else 0,
                "G": rinfo["G"], "W": rinfo["W"], "regs": rinfo["regs"], "ctas_per_sm": rinfo["ctas_per_sm"],
                "table": rinfo.get("table", "smem")}
        flops = 2.0 * K ** 3 * nsteps * b_local
        dmma = nt * (2 * nh * nh - (nh if (skip and nh == nt) else 0))  # DMMA.8x8x4 per segment-step
        extra = {"algorithm": "run-absorbing chain: absent runs applied as precomputed (Gamma Q)^r, r <= R",
                 "R": R, "steps": nsteps * b_local, "steps_per_record": nsteps / max(n_local, 1),
                 "executed_dmma_tflops": dmma * 512.0 * nsteps * b_local / (chain_avg / 1e3) / 1e12,
                 "reference_equivalent_tflops": 2.0 * K ** 3 * n_local * b_local / (chain_avg / 1e3) / 1e12,
                 "note": "achieved = 2K^3 per step / chain time; reference_equivalent counts 2K^3 per record "
                         "(the record-by-record algorithm's work) over the same time"}
    achieved = flops / (dom_ms / 1e3) / 1e12
    traffic = None
    for tname in ("r2_traffic.json", "r1_traffic.json"):
        tpath = os.path.join(ROOT, "profiles", tname)
        if traffic is None and os.path.exists(tpath):
            for t in json.load(open(tpath)).get("entries", []):
                if (t["workload"] == name and t["precision"] == args.precision
                        and t.get("path", "runs" if t.get("kernel", "").startswith("chain_runs") else "matrix")
                        == {2: "stitch", 1: "collapse"}.get(pmode, "runs" if runs else "matrix")):
                    traffic = (t["dram_read"] + t["dram_write"]) * n_local / t["n"]
                    if "dmma_pipe_active" in t:  # the shared FP64 pipe's occupancy in the same capture
                        extra = {**extra, "ncu_pipe_active": {"dmma": t["dmma_pipe_active"],
                                                              "fp64_simt": t["fp64_simt_pipe_active"],
                                                              "source": tname}}
                    break
    peak_src = "measured FP64 DMMA m8n8k4 microbenchmark, profiles/r1_fp64_peak_microbench.txt"
    if pmode in (1, 2):
        peak = FP64_DMMA_PEAK_TFLOPS
    elif runs:
        peak = FP64_DMMA_PEAK_TFLOPS
        kernel = f"chain_runs_kernel<nt={plan['nt']}, skip={int(skip and plan['tail'] == 0)}, tail={plan['tail']}> (R={R})"
    elif args.precision == "float64":
        peak = FP64_DMMA_PEAK_TFLOPS
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
    # achieved/frac: max over ranks of the dominant kernel's time (the slowest rank bounds the step)
    dom_max = ctx.reduce(dom_ms, "max")
    roofline = {"bound": "tensor", "achieved": achieved * dom_ms / dom_max, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved * dom_ms / dom_max / peak, "traffic": traffic, "kernel_ms": dom_ms,
                "traffic_note": "bytes/launch from the committed ncu capture (profiles/r*_traffic.json), "
                                "scaled to this launch's records; algorithmic 17 B/record",
                "kernel": kernel, "plan": plan, "peak_source": peak_src,
                "flops_per_launch": flops, "chain_ms": chain_avg, "fold_ms": statistics.mean(fold_ms),
                "chain_share_of_step": chain_avg / ms_per_step, "segments": nseg, **extra}
    _native.profile_enable(False)  # the e2e legs are timed on the host clock

    # ---- parity of the timed result vs the reference golden --------------
    want = golden_loglik(name, n_total) if args.precision == "float64" else None
    parity = float(np.max(np.abs(np.asarray(vals) - want) / np.abs(want))) if want is not None else None

    # ---- e2e through the public API from host arrays ----------------------
    pbytes = B * (K * K + 9 * K) * 8
    if use_dist and mode == "chain":
        host_pg = tuple(np.ascontiguousarray(a[lo_r:hi_r]) for a in (pr, lo, la))
        pin = [torch.from_numpy(np.ascontiguousarray(a.view(np.uint8) if a.dtype == np.bool_ else a)).pin_memory()
               .numpy() for a in host_pg]
        host_pin = (pin[0].view(np.bool_), pin[1], pin[2])
        fn_pg = lambda: sharded.loglik_batch(plist, cfg, stream=sptr, host_shard=host_pg)  # noqa: E731
        fn_pin = lambda: sharded.loglik_batch(plist, cfg, stream=sptr, host_shard=host_pin)  # noqa: E731
        api = "ShardedLoglik.loglik_batch(host_shard=...) (this rank's records from host memory)"
    elif use_dist:
        pin = [torch.from_numpy(np.ascontiguousarray(a.view(np.uint8) if a.dtype == np.bool_ else a)).pin_memory()
               .numpy() for a in (pr, lo, la)]
        host_pin = (pin[0].view(np.bool_), pin[1], pin[2])
        fn_pg = lambda: replica.loglik_batch(plist, cfg, stream=sptr, host=(pr, lo, la))  # noqa: E731
        fn_pin = lambda: replica.loglik_batch(plist, cfg, stream=sptr, host=host_pin)  # noqa: E731
        api = "ReplicaLoglik.loglik_batch(host=...)"
    else:
        pin = [torch.from_numpy(np.ascontiguousarray(a.view(np.uint8) if a.dtype == np.bool_ else a)).pin_memory()
               .numpy() for a in (pr, lo, la)]
        host_pin = (pin[0].view(np.bool_), pin[1], pin[2])
        if B > 1:
            fn_pg = lambda: eng.parallel_loglik_batch(plist, (pr, lo, la), cfg)  # noqa: E731
            fn_pin = lambda: eng.parallel_loglik_batch(plist, host_pin, cfg)  # noqa: E731
            api = "paper_2003_03508_b200.parallel_loglik_batch(params_list, (present, lon, lat), cfg)"
        else:
            fn_pg = lambda: eng._parallel_loglik_arrays(plist[0], pr, lo, la, cfg)  # noqa: E731
            fn_pin = lambda: eng._parallel_loglik_arrays(plist[0], *host_pin, cfg)  # noqa: E731
            api = "paper_2003_03508_b200._parallel_loglik_arrays(params, present, lon, lat, cfg)"
    h2d = n_local * 17 + pbytes
    e2e_pg_s, n_pg, first_pg = time_host_leg(ctx, fn_pg, ms_per_step, args.e2e_steps, f"{name} pageable")
    e2e_pin_s, n_pin, _ = time_host_leg(ctx, fn_pin, ms_per_step, args.e2e_steps, f"{name} pinned")
    autopin = os.environ.get("THMM_AUTOPIN", "1") != "0"
    e2e = {"value": B * n_total / e2e_pg_s, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
           "d2h_bytes_per_step": int(B * 12), "ms_per_step": e2e_pg_s * 1e3, "steps": n_pg, "api": api,
           "host_arrays": "pageable numpy (what the reference MCMC driver passes every call, bayes.py:712-715)",
           "transfer": ("the caller's pageable arrays are page-locked in place on first use (thmm_host_register; "
                        "released with the arrays), then read by the chain kernels over PCIe every call "
                        "(uncached loads, zero-copy); parameters H2D, result D2H" if autopin else
                        "H2D copy of the records in chunks on a copy stream, each chunk's chain launched behind "
                        "its copy (copies overlap the chain); parameters H2D, result D2H"),
           "first_call_ms": first_pg * 1e3,
           "pinned": {"value": B * n_total / e2e_pin_s, "unit": UNIT, "ms_per_step": e2e_pin_s * 1e3,
                      "steps": n_pin, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(B * 12),
                      "transfer": "zero-copy: the chain kernels read the pinned arrays in place over PCIe every "
                                  "call (uncached ld.global.cv, coordinates of present records only)"}}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            cpu = cpu_rate(plist[:1], pr, lo, la, budget_s=12.0 if main else 6.0)
            cpu.pop("sample_records", None)
        except Exception as exc:  # pragma: no cover
            cpu = {"error": repr(exc)}
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
    n_locals = ctx.gather(int(n_local))
    if mode == "chain" and use_dist:
        if getattr(sharded, "combine_used", None) == "stitched":
            par = (f"chain-sharded x{world} (stitched combine: NCCL all-gather of each rank's final forward row + "
                   f"log-scale, then of the B inter-rank link terms)")
        else:
            par = (f"chain-sharded x{world} ({'peer-memory mailbox over NVLink' if transport_used == 'peer' else 'NCCL all-gather of range nodes'})")
    elif use_dist:
        par = f"proposal-sharded x{world} (NCCL all-gather of B logL values)"
    else:
        par = "1 GPU"
    out = {"value": value, "ms_per_step": ms_per_step, "steps": steps, "warmup": warmup,
           "scaling": (args.scaling if B == 1 else "strong"),
           "dtype": {"float64": "f64", "float32": "f32"}.get(args.precision, args.precision),
           "config": config_dict(name, world, args.scaling),
           "run": {"parallelism": par, "transport_used": transport_used,
                   "combine": getattr(sharded, "combine_used", None) if sharded is not None else None,
                   "N_per_gpu": n_local,
                   "n_local_per_rank": n_locals, "batch_per_gpu": b_local, "segments_per_gpu": nseg,
                   "synth_s": t_syn},
           "roofline": roofline, "e2e": e2e, "cpu_baseline": cpu, "clocks": clocks, "gpu_launches": launches,
           "parity_max_rel_vs_reference": parity,
           "parity_note": ("max relative deviation of the timed evaluation's logL from the reference engine's "
                           "golden (tests/golden/bench_configs.json)" if want is not None else
                           "no golden for this N")}
    if host_prop:
        out["host_proposal_pack"] = host_prop
    for h in (dev, sharded, replica):
        if h is not None:
            h.close()
    del pin, host_pin
    return out


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
    ctx = Ctx(world, rank, local, use_dist)
    res = measure(ctx, args, args.workload, args.steps, args.warmup, main=True)
    subs = {}
    names = [] if args.subconfigs in ("", "none") else [s for s in args.subconfigs.split(",") if s != args.workload]
    for name in names:
        r = measure(ctx, args, name, args.sub_steps, 3, main=False)
        subs[name] = {k: r[k] for k in ("value", "ms_per_step", "steps", "warmup", "scaling", "config", "run",
                                         "roofline", "e2e", "cpu_baseline", "clocks", "gpu_launches",
                                         "parity_max_rel_vs_reference") if k in r}
        if "host_proposal_pack" in r:
            subs[name]["host_proposal_pack"] = r["host_proposal_pack"]
    if rank == 0:
        line = {
            "metric": METRIC, "value": res["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": res["ms_per_step"], "higher_is_better": True,
            "scaling": res["scaling"], "vs_baseline": None, "dtype": res["dtype"],
            "data": "synthetic (reference bench recipe: prior draw + simulate_path, seeded; "
                    "paper_2003_03508_b200/synth.py)",
            "config": res["config"], "run": res["run"],
            "roofline": res["roofline"], "cpu_baseline": res["cpu_baseline"], "e2e": res["e2e"],
            "clocks": res["clocks"], "gpu_launches": res["gpu_launches"],
            "parity_max_rel_vs_reference": res["parity_max_rel_vs_reference"],
            "parity_note": res["parity_note"],
            **({"host_proposal_pack": res["host_proposal_pack"]} if "host_proposal_pack" in res else {}),
            "subconfigs": subs,
        }
        if "k25_n1e6_b256" in subs:
            be = subs["k25_n1e6_b256"]["e2e"]
            line["e2e"]["batch_b256"] = {k: be[k] for k in ("value", "unit", "ms_per_step", "h2d_bytes_per_step",
                                                             "d2h_bytes_per_step", "api", "host_arrays")}
            line["e2e"]["batch_b256"]["pinned_value"] = be["pinned"]["value"]
    # NCCL_DEBUG=INFO (set by the launcher) prints communicator lines at init
    # and teardown: the JSON line is printed between two barriers so no other
    # rank's teardown output can interleave with it.
    ctx.barrier()
    if rank == 0:
        print(json.dumps(line), flush=True)
    ctx.barrier()
    if use_dist:
        ctx.dist.destroy_process_group()


if __name__ == "__main__":
    main()
