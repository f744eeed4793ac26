"""Per-pass times of the 1024^3 solve as it runs (forward axes 0, 1, 2 with the spectral divide
fused into the axis-2 pass, backward axes 0, 1, 2), plus the whole solve and the 1024^3 complex
propagate's phase pass; CUDA events on the context stream."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2605_20491_b200 import api as A


def timed(ctx, fn, reps=3):
    fn()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(ctx.stream)
    for _ in range(reps):
        fn()
    e1.record(ctx.stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ctx = A.Context(0)
    n = int(os.environ.get("N", "1024"))
    grid = A.Grid.sem(8.0, (n + 1) // 5, 5, 3)
    op = grid.separable_operator(ctx, [lambda t: t * t] * 3)
    N = grid.node_count()
    b = A.splitmix_uniform(ctx, 1, N)
    y = torch.empty_like(b)
    res = {"n": n}
    seq = [(0, True, "store"), (1, True, "store"), (2, True, "div"),
           (0, False, "store"), (1, False, "store"), (2, False, "store")]
    res["per_pass_ms"] = [timed(ctx, lambda a=a, f=f, e=e: op.transform_pass_ex(b, a, f, e, out=y))
                          for a, f, e in seq]
    res["solve_ms"] = timed(ctx, lambda: op.solve(b, out=y))
    res["sum_pass_ms"] = sum(res["per_pass_ms"])
    res["tflops_solve"] = 12.0 * n ** 4 / (res["solve_ms"] * 1e-3) / 1e12
    if os.environ.get("CPLX", "1") == "1":
        del b, y
        torch.cuda.empty_cache()
        psi = torch.view_as_complex(A.splitmix_uniform(ctx, 7, 2 * N).view(-1, 2))
        o = torch.empty_like(psi)
        res["cplx_pass_ms"] = [timed(ctx, lambda a=a, f=f, e=e: op.transform_pass_ex(
            psi, a, f, e, dt=0.01, out=o), reps=2) for a, f, e in
            [(0, True, "store"), (1, True, "store"), (2, True, "phase"), (2, False, "store")]]
        res["propagate_ms"] = timed(ctx, lambda: op.propagate(psi, 0.01, out=o), reps=2)
    print(json.dumps(res))


main()
