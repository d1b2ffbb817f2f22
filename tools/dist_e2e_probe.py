"""World-1 sharded evaluation from host arrays (the bench's N>1 e2e leg) per
exchange transport, next to the single-GPU host-array entry.

    python tools/dist_e2e_probe.py
"""
import os
import socket
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2003_03508_b200 as eng  # noqa: E402
from paper_2003_03508_b200 import synth  # noqa: E402
from paper_2003_03508_b200.distributed import ShardedLoglik  # noqa: E402

with socket.socket() as s:
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
plist, pr, lo, la = synth.make_workload("k25_n1e6")
pin = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy() for a in (pr.view(np.uint8), lo, la)]
pin[0] = pin[0].view(np.bool_)
cfg = eng.EngineConfig()


def t(fn, reps=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


print(f"single-GPU _parallel_loglik_arrays: {t(lambda: eng._parallel_loglik_arrays(plist[0], *pin, cfg)):.3f} ms")
for tr in ("peer", "nccl"):
    sh = ShardedLoglik(pr, lo, la, device=0, transport=tr)
    sh.loglik_batch(plist, cfg)
    print(f"{tr:5s} device-resident:   {t(lambda: sh.loglik_batch(plist, cfg)):.3f} ms")
    print(f"{tr:5s} host shard:        {t(lambda: sh.loglik_batch(plist, cfg, host_shard=tuple(pin))):.3f} ms")
    sh.close()
dist.destroy_process_group()
