import os, sys, socket
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np
import fixtures as fx
import torch, torch.distributed as dist
import paper_2003_03508_b200 as eng
from paper_2003_03508_b200 import _native
from paper_2003_03508_b200.distributed import ShardedLoglik
with socket.socket() as s:
    s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
dist.init_process_group("gloo", rank=0, world_size=1)
rng = np.random.default_rng(7)
plist = [fx.random_params(rng, 25)]
pr, lo, la = fx.random_obs_arrays(rng, 30000, present_prob=0.3)
for mode in (0, 1):
    _native.set_collapse_mode(mode)
    sh = ShardedLoglik(pr, lo, la, device=0, transport="peer")
    stream = torch.cuda.Stream()
    a = sh._peer_loglik if False else None
    out = sh.loglik_batch(plist, eng.EngineConfig(), stream=stream.cuda_stream)
    print("mode", mode, "used", sh.transport_used, out)
    # direct comparisons
    from paper_2003_03508_b200 import _native as nat
    sh2 = ShardedLoglik(pr, lo, la, device=0, transport="nccl")
    print("  nccl", sh2.loglik_batch(plist, eng.EngineConfig(), stream=stream.cuda_stream))
    dev = eng.DeviceObservations(pr, lo, la)
    print("  dev ", dev.loglik_batch(plist, eng.EngineConfig()))
    sh.close(); sh2.close(); dev.close()
dist.destroy_process_group()
