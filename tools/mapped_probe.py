"""One zero-copy evaluation of the K=25 N=10^6 workload from pinned host
arrays (the e2e leg's call), for an ncu capture of the chain kernel's
system-memory (PCIe) traffic:

    ncu -k regex:chain_runs --metrics lts__t_sectors_aperture_sysmem_op_read.sum,\
dram__bytes_read.sum,gpu__time_duration.sum python tools/mapped_probe.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2003_03508_b200 as eng  # noqa: E402
from paper_2003_03508_b200 import synth  # noqa: E402

plist, pr, lo, la = synth.make_workload("k25_n1e6")
pin = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in (pr.view(np.uint8), lo, la)]
ppr, plo, pla = pin[0].numpy().view(np.bool_), pin[1].numpy(), pin[2].numpy()
for _ in range(3):
    v = eng._parallel_loglik_arrays(plist[0], ppr, plo, pla, eng.EngineConfig())
present = int(pr.sum())
print(f"logL {v:.10f}; records {pr.size}, present {present}; bytes: flags {pr.size}, "
      f"coordinates of present records {16 * present}")
