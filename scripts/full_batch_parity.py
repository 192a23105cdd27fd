"""Every env of the N=10 bench batches (131,072 envs: MT and arctic, BASELINE configs[4]'s per-GPU
share) against the reference stepping all of them (WorkerPool over every host core), across an
episode boundary -- the full-batch counterpart of tests/test_gpu_scale.py's 768-env samples.
Usage: python scripts/full_batch_parity.py [task:N:B:steps] ..."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import refbind as ref  # noqa: E402
from scale_parity import run_full_batch  # noqa: E402
from test_gpu_step import make_cfgs  # noqa: E402

args = sys.argv[1:] or ["material_transport:10:131072:75", "arctic_transport:10:131072:105"]
for a in args:
    task, n, B, steps = a.split(":")
    cfg, sp = make_cfgs(ref, task, int(n))
    rep = run_full_batch(ref, cfg, sp, int(B), int(steps), every=15)
    rep["task"], rep["N"] = task, int(n)
    print(json.dumps(rep, default=str), flush=True)
