"""Config-5 9D n = 9 kinetic propagate (Kronecker path), CUDA events on the context stream;
variant libraries via KRONOP_LIB. Prints ms per propagate and a checksum."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2605_20491_b200 import api as A

ctx = A.Context(0)
dims = sys.argv[1:] or ["9d"]
res = {"lib": os.path.basename(os.environ.get("KRONOP_LIB", "default"))}
for name in dims:
    L, cells, k, d = {"9d": (3.0, 2, 5, 9), "6d": (5.0, 3, 10, 6)}[name]
    g = A.Grid.sem(L, cells, k, d)
    lap = g.laplacian(ctx)
    psi = torch.view_as_complex(A.splitmix_uniform(ctx, 3, 2 * g.node_count()).view(-1, 2))
    o = torch.empty_like(psi)
    lap.propagate(psi, 0.005, out=o)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(ctx.stream)
    for _ in range(5):
        lap.propagate(psi, 0.005, out=o)
    e1.record(ctx.stream)
    torch.cuda.synchronize()
    res[name + "_propagate_ms"] = e0.elapsed_time(e1) / 5
    res[name + "_checksum"] = float(torch.view_as_real(o).abs().sum())
    del psi, o, lap
    torch.cuda.empty_cache()
print(json.dumps(res))
