

timeout 900 ncu --set full --clock-control none -k "regex:mode_product_tma_kernel<.*, 6>" -c 1 -o /tmp/r02_split python -c "
import torch
from paper_2605_20491_b200 import api as A, slab as S
ctx = A.Context(0)
g = A.Grid.sem(8.0, 205, 5, 3)
op = g.separable_operator(ctx, [lambda t: t * t] * 3)
so = S.DeviceSlabOperator(op.axes, devices=[0, 0])
b = A.splitmix_uniform(ctx, 1, g.node_count())
bs = so.scatter(b)
x = so.solve(bs)
torch.cuda.synchronize()
" > /tmp/b.log 2>&1
python tools/ncu_summary.py /tmp/r02_split.ncu-rep gpurun_out/r02_split_pass.json > /dev/null
cat gpurun_out/r02_kron9_pair.json gpurun_out/r02_split_pass.json | grep -E "kernel|duration|dram|pipe"
