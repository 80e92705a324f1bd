#!/usr/bin/env python
"""Train and commit a model for a bench workload (run on a GPU box; off the hot path).

    python scripts/train_model.py --workload acl-512k --model paper --seconds 300

Labels come from train.torch_labels (a plain torch brute-force scan, no libtang), on a training
trace drawn with seed 7 (uniform), so nothing the oracle consumes passes through the CUDA
library.  Writes models/<workload>_<model>.npz (tang_inputs.save_model: W1/W2/Wo rounded to bf16, W0/biases fp32) with the
training metadata; bench.py and the full-size parity test load it."""
import argparse
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402  (workload table)
import tang_inputs as ti  # noqa: E402
from paper_2601_03187_b200 import train as TR  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="acl-512k")
ap.add_argument("--model", default="paper")
ap.add_argument("--seconds", type=float, default=300.0)
ap.add_argument("--packets", type=int, default=1 << 22)
ap.add_argument("--out", default=None)
a = ap.parse_args()
fam, n_rules, seed, kind = bench.WORKLOADS[a.workload]
N, B = bench.MODELS[a.model]
rules = ti.classbench_ruleset(fam, n_rules, seed)
sigs = TR.tuple_signatures(rules)
tr = ti.uniform_trace(rules, a.packets, 7) if kind == "uniform" else np.concatenate(
    [ti.uniform_trace(rules, a.packets // 2, 7), ti.zipf_trace(rules, a.packets - a.packets // 2, 8, perm_seed=seed)])
d = torch.from_numpy(tr.view(np.uint8).copy()).cuda()
t0 = time.time()
labels = TR.torch_labels(rules, sigs, d)
print(f"labels: {time.time() - t0:.1f}s, unmatched {(labels < 0).float().mean().item():.4f}", flush=True)
w, acc = TR.train(rules, sigs, N, B, d, labels, seconds=a.seconds, log=lambda *m: print(*m, flush=True))
meta = dict(workload=a.workload, model=a.model, rules=int(rules.size), ruleset_seed=seed, trace_seed=7,
            train_packets=a.packets, seconds=a.seconds, train_accuracy=acc, labels="train.torch_labels",
            command=" ".join(sys.argv), torch=torch.__version__)
out = a.out or ti.model_path(a.workload, a.model)
os.makedirs(os.path.dirname(out), exist_ok=True)
ti.save_model(out, sigs, TR.round_weights_bf16(w), meta)
print(f"wrote {out}: N={N} B={B} C={len(sigs)} train acc {acc:.4f}", flush=True)
