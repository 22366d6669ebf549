"""Harness: stress the single-launch small-matrix kernel (default 4x2 cluster): many back-to-back
evaluations of several plans, every result compared bit for bit with the first."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_11843_b200 as P  # noqa: E402
from paper_2602_11843_b200 import inputs  # noqa: E402

h = P.nseries_create(0)
n = int(os.environ.get("STRESS_N", "20000"))
bad = 0
for steps, k, fl in (([9, 9], 81, 0), ([15, 15], 225, P.NSERIES_ALLOW_APPROX), ([5, 1, 9], 54, 0)):
    for d in (64, 37):
        A = torch.from_numpy(inputs.random_matrix(d, 3, 0.6)).cuda()
        plan = P.nseries_plan_finalize(steps, k, fl)
        outs = [torch.empty_like(A) for _ in range(8)]
        P.nseries_eval(h, A, d, k, plan=plan, S=outs[0], flags=fl)
        torch.cuda.synchronize()
        ref = outs[0].clone()
        for i in range(n // 6):
            o = outs[i % 8]
            P.nseries_eval(h, A, d, k, plan=plan, S=o, flags=fl)
            if i % 8 == 7:
                torch.cuda.synchronize()
                for x in outs:
                    bad += int(not torch.equal(x, ref))
        torch.cuda.synchronize()
        print(steps, d, "mismatches so far", bad, flush=True)
print("done, mismatches:", bad)
