"""Time single mode-product passes (kronop_op_pass) for each axis at a few sizes; used to compare
kernel variants (KRONOP_LIB=<variant .so>)."""
import json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2605_20491_b200 import api as A

def main():
    res = {"lib": os.environ.get("KRONOP_LIB", "default")}
    ctx = A.Context(0)
    cfgs = {1024: (205, 5), 512: (27, 19), 499: (100, 5), 79: (8, 10), 64: (13, 5)}
    which = os.environ.get("PASS_CASES", "1024r,1024c,512r,499c,79r,64r").split(",")
    for case in which:
        n, cplx = int(case[:-1]), case[-1] == "c"
        cells, k = cfgs[n]
        grid = A.Grid.sem(8.0, cells, k, 3)
        op = grid.separable_operator(ctx, [lambda t: t * t] * 3)
        N = grid.node_count()
        x = A.splitmix_uniform(ctx, 1, 2 * N if cplx else N)
        if cplx:
            x = torch.view_as_complex(x.view(-1, 2))
        y = torch.empty_like(x)
        nn = grid.shape[0]
        times = []
        for axis in range(3):
            for _ in range(2):
                op.transform_pass(x, axis, True, out=y)
            reps = max(3, int(2e11 / (2 * nn * N)))
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(ctx.stream)
            for _ in range(reps):
                op.transform_pass(x, axis, True, out=y)
            e1.record(ctx.stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1) / reps)
        fl = 2.0 * nn * N * (2 if cplx else 1)
        res["n%d%s" % (nn, "c" if cplx else "")] = {"ms": times, "tflops": [fl / (t * 1e-3) / 1e12 for t in times]}
        del x, y, op
        torch.cuda.empty_cache()
    print(json.dumps(res))

main()
