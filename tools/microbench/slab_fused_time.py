"""1024^3 solve on P virtual slabs (one GPU, P streams): exchange-fused transposes vs the copy
exchange (run twice, KRONOP_SLAB_FUSED=0 for the second), CUDA events over all parts' streams."""
import json, os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2605_20491_b200 import api as A, slab as S

ctx = A.Context(0)
grid = A.Grid.sem(8.0, 205, 5, 3)
op = grid.separable_operator(ctx, [lambda t: t * t] * 3)
b = A.splitmix_uniform(ctx, 1, grid.node_count())
res = {"fused_env": os.environ.get("KRONOP_SLAB_FUSED", "1")}
for P in (1, 2, 4):
    so = S.DeviceSlabOperator(op.axes, devices=[0] * P)
    bs = so.scatter(b)
    xs = so.solve(bs)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        xs = so.solve(bs)
    torch.cuda.synchronize()
    res["P%d_ms" % P] = (time.perf_counter() - t0) / 3 * 1e3
    res["P%d_fused" % P] = so.fused_transforms()
    del bs, xs
    so.close()
    torch.cuda.empty_cache()
print(json.dumps(res))
