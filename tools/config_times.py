"""Device time of one evaluation for every BASELINE config (c1-c5) through the
C ABI (CUDA events, after warm-up).  Not the bench contract (bench.py is c5);
a survey of where each config stands.  python tools/config_times.py [--reps R]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import dvm_inputs  # noqa: E402
from paper_1201_3986_b200 import Plan  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--c5cells", type=int, default=36)
args = ap.parse_args()
out = {}
for name in ("c1", "c2", "c3", "c4", "c5"):
    cfg = dvm_inputs.CONFIGS[name]
    cells = args.c5cells if name == "c5" else None
    f = torch.from_numpy(dvm_inputs.make(name, cells=cells) if cells else dvm_inputs.make(name)).cuda()
    p = Plan(cfg.d, cfg.N, cfg.Nbar)
    q = torch.empty_like(f)
    for _ in range(3):
        p.collide(f, q)
    reps = 2 if name == "c5" else args.reps
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(reps):
        p.collide(f, q)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    p.profile(True)
    p.collide(f, q)
    prof = {k: round(v[0], 4) for k, v in p.profile_read().items() if v[1]}
    p.profile(False)
    ncell = f.shape[0]
    nodes = cfg.N ** cfg.d
    eff = (p.A + 2) * 8.0 * nodes * ncell / (ms / 1e3) / 1e9  # streaming formulation, SURVEY 8(d)
    out[name] = {"ms_per_eval_batch": ms, "cells": ncell, "evals_per_s": ncell / (ms / 1e3), "A": p.A,
                 "Ntilde": p.Ntilde, "effective_streaming_GBps": eff, "kernels_ms": prof}
    print(name, json.dumps(out[name]), flush=True)

