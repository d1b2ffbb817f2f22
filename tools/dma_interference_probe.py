import os, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2003_03508_b200 as eng
from paper_2003_03508_b200 import _native, synth
plist, pr, lo, la = synth.make_workload("k80_n1e8", n=20_000_000)
dev = eng.DeviceObservations(pr, lo, la)
cfg = eng.EngineConfig()
p = plist[0]
for _ in range(3): dev.loglik(p, cfg)
def t(reps=10):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): dev.loglik(p, cfg)
    return (time.perf_counter() - t0) / reps * 1e3
print("alone", t())
h = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)
d = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(40): d.copy_(h, non_blocking=True)
print("with concurrent 1 GB H2D copies", t())
torch.cuda.synchronize()
with torch.cuda.stream(s):
    for _ in range(40): d.copy_(d.flip(0) if False else h, non_blocking=True)
print("again", t())
torch.cuda.synchronize()
print("alone", t())
