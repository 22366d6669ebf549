"""Harness: bit-determinism of repeated fp32 evaluations (split-K tail tiles), per d.
Mirrors tests/test_gpu_parity.py::_run (NaN-filled S, plan from nseries_plan_finalize)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_11843_b200 import _binding as P, inputs  # noqa: E402

h = P.nseries_create(0)
for d in [int(x) for x in os.environ.get("DET_D", "1024,1100,1500,2100").split(",")]:
    A = torch.from_numpy(inputs.random_matrix(d, 77, 0.9).astype(np.float32)).cuda()
    plan = P.nseries_plan_finalize([9, 9], 81, 0)
    outs = []
    for r in range(3):
        S = torch.full_like(A, float("nan"))
        P.nseries_eval(h, A, d, 81, plan=plan, S=S)
        torch.cuda.synchronize()
        outs.append(S.cpu().numpy())
    for r in range(3):
        nan = np.argwhere(np.isnan(outs[r]))
        if len(nan):
            print(d, "run", r, "NaN", len(nan), "rows", nan[:, 0].min(), nan[:, 0].max(), "cols", nan[:, 1].min(),
                  nan[:, 1].max(), flush=True)
    for r in (1, 2):
        diff = np.argwhere(~((outs[0] == outs[r]) | (np.isnan(outs[0]) & np.isnan(outs[r]))))
        print(d, r, "ndiff", len(diff), diff[:3].tolist(), flush=True)
