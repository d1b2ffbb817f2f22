"""Host side of the e2e leg: H2D bandwidth of the 17 MB record upload and the
pipelined host-array evaluation, with the process on all CPUs vs pinned to
the GPU's NUMA-local CPUs (pinned buffers first-touched after the pin).

    python tools/host_affinity_probe.py
"""
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2003_03508_b200 as eng  # noqa: E402
from paper_2003_03508_b200 import synth  # noqa: E402


def sh(cmd):
    try:
        return subprocess.run(cmd, shell=True, capture_output=True, text=True, timeout=30).stdout
    except Exception as exc:  # noqa: BLE001
        return str(exc)


print(sh("nvidia-smi topo -m"))
print(sh("lscpu | grep -i -E 'numa|model name|socket|^CPU\\(s\\)'"))
bus = torch.cuda.get_device_properties(0).pci_bus_id if hasattr(torch.cuda.get_device_properties(0), "pci_bus_id") else None
print("pci bus", bus)

plist, pr, lo, la = synth.make_workload("k25_n1e6")
p = plist[0]
cfg = eng.EngineConfig()


def pinned():
    out = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy() for a in (pr.view(np.uint8), lo, la)]
    out[0] = out[0].view(np.bool_)
    return out


def t(fn, reps=100):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


def run(tag):
    pin = pinned()
    dev = eng.DeviceObservations(*pin)
    h = torch.empty(17_000_000, dtype=torch.uint8).pin_memory()
    d = torch.empty_like(h, device="cuda")
    bw = 17e6 / t(lambda: d.copy_(h, non_blocking=True)) / 1e6
    print(f"[{tag}] raw H2D 17 MB: {bw:.1f} GB/s")
    print(f"[{tag}] loglik device-resident:  {t(lambda: dev.loglik(p, cfg)):.3f} ms")
    print(f"[{tag}] _parallel_loglik_arrays: {t(lambda: eng._parallel_loglik_arrays(p, *pin, cfg)):.3f} ms", flush=True)


run("all cpus")
node_cpus = None
try:
    from pynvml import nvmlInit, nvmlDeviceGetHandleByIndex, nvmlDeviceGetCpuAffinity
    nvmlInit()
    mask = nvmlDeviceGetCpuAffinity(nvmlDeviceGetHandleByIndex(0), 16)
    node_cpus = [w * 64 + b for w, m in enumerate(mask) for b in range(64) if m >> b & 1]
except Exception as exc:  # noqa: BLE001
    print("nvml affinity unavailable:", exc)
print("gpu-local cpus:", node_cpus)
if node_cpus:
    os.sched_setaffinity(0, node_cpus)
    run("gpu-local cpus")
