"""A/B of the spectral launch of the small-extent (fused_rot) path: KRONOP_ROT_SPEC_SPLIT = 0 (epilogue
fused into the 16-warp DMMA contraction), 1 (split when the DFMA kernel serves the group, default),
2 (split for every extent). Each mode runs in its own process (the switch is read once); prints the
per-propagate / per-solve times and a digest of the outputs, which must agree bit for bit.

  python tools/microbench/spec_split.py            # driver: runs the three modes, one JSON line
  python tools/microbench/spec_split.py --child    # one mode (env) -> JSON
"""
import hashlib
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def child():
    import torch
    sys.path.insert(0, ROOT)
    from paper_2605_20491_b200 import api as A
    ctx = A.Context(0)
    res = {}
    for name, (L_, cells, k, d) in {"6d_n29": (5.0, 3, 10, 6), "9d_n9": (3.0, 2, 5, 9)}.items():
        g = A.Grid.sem(L_, cells, k, d)
        lap = g.laplacian(ctx)
        N = g.node_count()
        psi = torch.view_as_complex(A.splitmix_uniform(ctx, 3, 2 * N).view(-1, 2))
        o = torch.empty_like(psi)
        for what in ("propagate", "solve"):
            if what == "propagate":
                run = lambda: lap.propagate(psi, 0.005, out=o)  # noqa: E731
                tgt = o
            else:
                u = torch.view_as_real(psi).reshape(-1)[:N].contiguous()
                ou = torch.empty_like(u)
                run = lambda: lap.solve(u, out=ou)  # noqa: E731
                tgt = ou
            run()
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(ctx.stream)
            for _ in range(5):
                run()
            e1.record(ctx.stream)
            torch.cuda.synchronize()
            dig = hashlib.sha1(tgt.view(torch.float64).cpu().numpy().tobytes()).hexdigest()[:16]
            res["%s_%s" % (name, what)] = {"ms": e0.elapsed_time(e1) / 5, "digest": dig}
            if what == "solve":
                del u, ou
        del lap, psi, o
        torch.cuda.empty_cache()
    print(json.dumps(res))


def main():
    out = {}
    for mode in ("0", "1", "2"):
        env = dict(os.environ, KRONOP_ROT_SPEC_SPLIT=mode)
        p = subprocess.run([sys.executable, os.path.abspath(__file__), "--child"], env=env,
                           capture_output=True, text=True, timeout=600)
        if p.returncode != 0:
            out["mode" + mode] = {"error": p.stderr[-400:]}
            continue
        out["mode" + mode] = json.loads(p.stdout.strip().splitlines()[-1])
    modes = [m for m in out.values() if "error" not in m]
    if modes:
        out["bitwise_equal"] = all(
            all(m[k]["digest"] == modes[0][k]["digest"] for k in modes[0]) for m in modes)
    print(json.dumps(out))


if __name__ == "__main__":
    child() if "--child" in sys.argv else main()
