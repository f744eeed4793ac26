"""In-box comparator: the three 1024^3 pass shapes of the solve as cuBLAS DGEMMs
(torch.matmul on float64 -> cublasDgemm / cublasDgemmStridedBatched), CUDA events, next to the
TMA/DMMA pass kernel's per-pass times (tools/microbench/solve_passes.py). Layout as the field:
axis 0 fastest.
  axis 0: Y (1024 x n^2) = A (1024 x 1024) X (1024 x n^2)              one DGEMM
  axis 1: Y_q = X_q A^T for the n slabs q (each 1024 x 1024)           strided batched, n batches
  axis 2: Y (n^2 x 1024) = X (n^2 x 1024) A^T                            one DGEMM
"""
import json
import torch

n = 1024
A = torch.randn(n, n, dtype=torch.float64, device="cuda")
X = torch.randn(n * n * n, dtype=torch.float64, device="cuda")
Y = torch.empty_like(X)


def t(fn, reps=3):
    fn()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


# torch tensors are row-major; the field (axis 0 fastest) of shape (n0, n1, n2) is the row-major
# array [n2][n1][n0].
x3 = X.view(n, n, n)   # [i2][i1][i0]
y3 = Y.view(n, n, n)
res = {}
# axis 0: y[i2][i1][:] = A x[i2][i1][:]  ->  (n^2 x n) @ A^T
res["axis0_ms"] = t(lambda: torch.matmul(X.view(n * n, n), A.t(), out=Y.view(n * n, n)))
# axis 1: for each i2: y[i2] (n1 x n0) = A @ x[i2]   -> batched (n, n, n)
res["axis1_ms"] = t(lambda: torch.matmul(A, x3, out=y3))
# axis 2: y (n x n^2) = A @ x (n x n^2)
res["axis2_ms"] = t(lambda: torch.matmul(A, X.view(n, n * n), out=Y.view(n, n * n)))
for k in ("axis0", "axis1", "axis2"):
    res[k + "_tflops"] = 2.0 * n ** 4 / (res[k + "_ms"] * 1e-3) / 1e12
res["solve_equiv_ms"] = 2 * (res["axis0_ms"] + res["axis1_ms"] + res["axis2_ms"])
print(json.dumps(res))
