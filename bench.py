"""Benchmark: (-Delta + V1)^{-1} apply at 1024^3 FP64 on B200 (BASELINE.json configs[1]).

One step = one SeparableOperator::solve (operators.cpp:42-61) of a 1024^3 real field: 3 forward
mode-product passes (T^{-1}), the fused spectral divide, 3 backward passes (T). SEM Q^5, 205 cells,
L = 8 (n = 1024), harmonic V1 = x^2 per axis, rhs = SplitMix64(seed = 1) uniform [-1, 1)
(harness.cpp:184-189). Fields are 8 GiB each (>> 126 MB L2), so no L2 flush is needed.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl kronop|reference] [--extent 1024]

--impl reference times the reference's CPU path on the host cores at the same 1024^3 workload (no
scaling): the C++ -O3 -fopenmp restatement of tensor.cpp / operators.cpp in oracle/cpu (the
reference itself cannot be built here, Eigen3 is absent), one full solve per step.
Multi-GPU (--gpus N self-launches torch.distributed.run; one rank per GPU): the same solve is
slab-decomposed through the C-ABI (kronop_slab_create_nccl, csrc/slab.cu): axes 0-1
local, two NCCL all-to-all transposes for the last axis; total work fixed => "scaling": "strong";
time = max over ranks of CUDA-event time. --extent 2048 selects the 2048^3 scaling grid (Q3 x 683).
"""
import argparse
import json
import math
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAK_FP64_FALLBACK = 35.4  # TFLOP/s, cuBLAS DGEMM sustained measured on this pool (profiles/)


def load_peaks():
    peaks = {"hbm_gbs": 6449.1, "fp64_tflops": PEAK_FP64_FALLBACK, "fp64_src": "fallback"}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        peaks["hbm_gbs"] = m.get("hbm_gbs", peaks["hbm_gbs"])
    except OSError:
        pass
    try:
        with open(os.path.join(ROOT, "profiles", "r01_fp64_dgemm_peak.json")) as f:
            m = json.load(f)
        peaks["fp64_tflops"] = m["fp64_tflops_sustained"]
        peaks["fp64_src"] = "measured cuBLAS DGEMM sustained (profiles/r01_fp64_dgemm_peak.json)"
    except (OSError, KeyError):
        pass
    return peaks


def load_pass_traffic():
    """DRAM bytes per 1024^3 pass of the dominant kernel from the committed `ncu --set full`
    capture of the current kernels (dram__bytes_read.sum + dram__bytes_write.sum of the first
    pass of the rotated solve -- the CONTIG TMA instance every pass of the solve runs,
    profiles/r02_rotated_pass.json; else the axis-order STRIDED pass, r02_pass_a1.json), else
    round 1's, else None."""
    def gb(v):
        return float(v.split()[0]) * {"Gbyte": 1e9, "Mbyte": 1e6, "Tbyte": 1e12}[v.split()[1]]
    for name in ("r02_rotated_pass.json", "r02_pass_a1.json"):
        try:
            with open(os.path.join(ROOT, "profiles", name)) as f:
                k = json.load(f)["kernels"][0]
            return gb(k["dram_read"]) + gb(k["dram_write"])
        except (OSError, KeyError, ValueError, IndexError):
            pass
    try:
        with open(os.path.join(ROOT, "profiles", "r01_ncu_full_pass1024.json")) as f:
            m = json.load(f)
        return m["traffic_bytes_per_launch"]
    except (OSError, KeyError, ValueError):
        return None


class ClockSampler:
    def __init__(self, gpu_index=0):
        self.proc = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(gpu_index),
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out = self.proc.communicate()[0]
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in out.strip().splitlines():
            p = [x.strip() for x in ln.split(",")]
            try:
                sm.append(float(p[0]))
                mx.append(float(p[1]))
            except (ValueError, IndexError):
                continue
            for nm, v in zip(names, p[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_init():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl")
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(world, v, device):
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def workload_config(n):
    """SEM cells of the workload family at extent n = cells * degree - 1 (basis1d.cpp:23,55):
    Q5 for the BASELINE 1024^3 config (205 cells), Q3 for the 2048^3 scaling grid (683 cells,
    SURVEY.md §8a C4)."""
    for k in (5, 3):
        if (n + 1) % k == 0:
            return (n + 1) // k
    raise SystemExit("n must be 5*cells - 1 or 3*cells - 1 (1024 = Q5 x 205, 2048 = Q3 x 683)")


def workload_degree(n):
    return 5 if (n + 1) % 5 == 0 else 3


# -------------------------------------------------------------------------- CPU arm --
def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_reference_operator(n):
    """The reference CPU path at the full workload: the C++ restatement of tensor.cpp /
    operators.cpp (oracle/cpu/kronop_cpu.cpp: zero-filled std::vector fields, OpenMP static
    partitions of single-threaded OpenBLAS GEMMs, serial spectral loop), on all host cores, with
    the oracle's axis factorisation (numpy build_axis; harmonic V1, so the three axes are equal)."""
    from oracle import kronop_oracle as K
    from oracle import kronop_cpu as KC
    # every host core, whatever OMP_NUM_THREADS a launcher set (torchrun sets 1 per rank)
    KC.lib(os.cpu_count() or 1)
    ax = K.build_axis(K.assemble_sem(8.0, workload_config(n), workload_degree(n)), lambda t: t * t)
    return KC, KC.CpuOperator([ax] * 3)


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return 0
    n = args.n
    N = n ** 3
    KC, co = cpu_reference_operator(n)
    b = KC.uniform_pm1(1, N)  # random_field(seed 1) (harness.cpp:184-189)
    # one solve takes ~20 s on 16 cores: the warm-up and timed counts are capped so the arm ends
    # in a few minutes; "steps" is the number actually timed (steps_requested: the driver's K)
    warm, steps = min(args.warmup, 1), max(1, min(args.steps, 3))
    if warm:
        KC.time_op(co, "solve", b, warm)
    _, secs = KC.time_op(co, "solve", b, steps)
    t = float(np.median(secs))
    gdofs = N / t / 1e9
    cores = KC.threads()
    sample = ("full %d^3 (-Delta+V1)^-1 solve (no scaling), C++ -O3 -fopenmp restatement of "
              "tensor.cpp/operators.cpp (OpenBLAS DGEMM per OpenMP chunk, serial spectral loop, "
              "zero-filled fields), median of %d after %d warm-up; %s" % (n, steps, warm, cpu_model()))
    line = {
        "impl": "reference", "metric": "(-Delta+V1)^-1 apply GDoF/s at 1024^3 fp64",
        "value": gdofs, "unit": "GDoF/s", "n_gpus": world, "steps": steps,
        "steps_requested": args.steps, "warmup": warm, "ms_per_step": t * 1e3,
        "step_ms": [round(x * 1e3, 1) for x in secs], "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "3D (-Delta+V1)^-1 solve, harmonic V1, SEM Q%d %d cells L=8, n=%d"
                               % (workload_degree(n), workload_config(n), n),
                   "n": n, "dof": N},
        "cpu_baseline": {"value": gdofs, "unit": "GDoF/s", "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": gdofs, "unit": "GDoF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def cpu_leg(n, b_host, x_gpu_host):
    """cpu_baseline of the GPU arm: one C++ reference-path solve of the same 1024^3 workload on the
    host cores (same rhs), its time, and the GPU solution's relative difference to it."""
    KC, co = cpu_reference_operator(n)
    xr, secs = KC.time_op(co, "solve", b_host, 1)
    rel = float(np.linalg.norm(x_gpu_host - xr) / np.linalg.norm(xr))
    mx = float(np.abs(x_gpu_host - xr).max() / np.abs(xr).max())
    return {"value": n ** 3 / secs[0] / 1e9, "unit": "GDoF/s", "cores": KC.threads(), "kind": "port",
            "sample": "one full %d^3 solve (no scaling), C++ -O3 -fopenmp restatement of the "
                      "reference CPU path (OpenBLAS DGEMM per OpenMP chunk), %s" % (n, cpu_model()),
            "seconds": secs[0], "rel_diff_vs_oracle": rel, "max_rel_diff_vs_oracle": mx}


# -------------------------------------------------------------------------- GPU arm --
def secondary_metrics(A, P, ctx, device):
    """The other two metrics BASELINE.json names, each timed on the device:
    PCG time-to-tol (stirrer, 512^3 = Q19 x 27 cells, seed-1 rhs, tol 1e-8, (-Delta+V1)^-1
    preconditioner; harness.cpp:501-582) and split-step steps/s (Strang = qHOP M=1 with merge,
    499^3 complex128, sep-osc trap split=kinetic, box psi0, dt = 5e-3, T = 0.1;
    splitting.cpp:107-146)."""
    import torch
    out = {}
    g = A.Grid.sem(8.0, 27, 19, 3)
    pot = P.build_potential("stirrer", g)
    op = g.separable_operator(ctx, pot.separable)
    v2 = pot.v2_device("cuda:%d" % device)
    b = A.splitmix_uniform(ctx, 1, g.node_count())
    x = torch.zeros_like(b)
    cfg = A.PcgConfig(rel_tol=1e-8)
    A.pcg(A.apply_map(op, v2), A.solve_map(op), b, x, A.PcgConfig(rel_tol=1e-8, max_iter=2))
    x.zero_()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(ctx.stream)
    rep = A.pcg(A.apply_map(op, v2), A.solve_map(op), b, x, cfg)
    e1.record(ctx.stream)
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 1e3
    n = g.shape[0]
    out["pcg_time_to_tol"] = {
        "value": t, "unit": "s", "iterations": rep.iterations, "final_residual": rep.final_residual,
        "converged": rep.converged, "n": n, "dof": g.node_count(),
        "tflops": (rep.iterations + 1) * 24.0 * n ** 4 / t / 1e12,
        "config": "stirrer V=V1+V2, SEM Q19 x 27 cells (n=512), L=8, rhs SplitMix64(1), tol 1e-8, "
                  "precond (-Delta+V1)^-1, device-resident PCG (one CUDA graph, WHILE node)"}
    try:  # variant: the same PCG with every transform on the INT8 path (kronop_op_set_precision)
        xd = x.clone()
        op.set_precision("ozaki")
        x.zero_()
        A.pcg(A.apply_map(op, v2), A.solve_map(op), b, x, A.PcgConfig(rel_tol=1e-8, max_iter=2))
        x.zero_()
        torch.cuda.synchronize()
        e0.record(ctx.stream)
        repo = A.pcg(A.apply_map(op, v2), A.solve_map(op), b, x, cfg)
        e1.record(ctx.stream)
        torch.cuda.synchronize()
        to = e0.elapsed_time(e1) / 1e3
        out["pcg_time_to_tol_ozaki"] = {
            "value": to, "unit": "s", "iterations": repo.iterations,
            "iterations_fp64": rep.iterations, "final_residual": repo.final_residual,
            "rel_diff_vs_fp64": float(torch.linalg.norm(x - xd) / torch.linalg.norm(xd)),
            "config": "variant of pcg_time_to_tol: the operator and the preconditioner on FP64 "
                      "emulated on the INT8 tensor cores (Ozaki, 7 slices), same graph-captured PCG"}
        op.set_precision("fp64")
        del xd
    except Exception as e:  # reported, never silently replaced
        out["pcg_time_to_tol_ozaki"] = {"error": str(e)[:200]}
    del op, v2, b, x
    torch.cuda.empty_cache()
    g = A.Grid.sem(8.0, 100, 5, 3)
    pot = P.build_potential("sep-osc", g, quad_coeffs=[1.0] * 3, osc_amplitude=100.0)
    lap = g.laplacian(ctx)
    bdiag = torch.from_numpy(np.array(P.separable_sum(g, pot))).to("cuda:%d" % device)
    box = g.sample(lambda c: np.sin(np.pi * (c[0] + 8.0) / 16.0) * np.sin(np.pi * (c[1] + 8.0) / 16.0)
                   * np.sin(np.pi * (c[2] + 8.0) / 16.0))
    psi0 = torch.from_numpy(box.astype(np.complex128)).to("cuda:%d" % device)
    spec = A.SplitSpec(quad_points=1, composition="single", dt=1e-3, total_time=0.1,
                       merge_across_steps=True)
    A.evolve(A.SplitSpec(quad_points=1, dt=1e-3, total_time=5e-3, merge_across_steps=True), lap,
             bdiag, psi0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    state, err, steps = A.evolve(spec, lap, bdiag, psi0)
    torch.cuda.synchronize()
    t = time.perf_counter() - t0
    # error against the exact propagator of the full separable H (splitting.cpp:127-141), untimed
    full = g.separable_operator(ctx, pot.separable)
    psi0n = psi0 / torch.linalg.norm(psi0)
    split_err = float(torch.linalg.norm(state - full.propagate(psi0n, 0.1)))
    del full, psi0n
    out["splitstep_steps_per_s"] = {
        "value": steps / t, "unit": "steps/s", "steps": steps, "seconds": t, "n": g.shape[0],
        "error_vs_exact": split_err, "paper_error": 5.21e-5,
        "config": "Strang (qHOP M=1) with cross-step merge, 499^3 complex128 (SEM Q5 x 100 cells, "
                  "L=8), A=-Delta, B=sep-osc V, box psi0, dt=1e-3, T=0.1: the PAPER.md:1378-1381 "
                  "row (M=1, dt=0.001: error 5.21e-5, 100 steps in 9.5 s on GH200)"}
    # the same run with the even/odd folded kinetic operator (-Delta on the symmetric SEM grid
    # commutes with x -> -x per axis): half the transform flops, same state to ~1e-12
    lapf = g.laplacian(ctx, folded=True)
    A.evolve(A.SplitSpec(quad_points=1, dt=1e-3, total_time=5e-3, merge_across_steps=True), lapf,
             bdiag, psi0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    statef, _, stepsf = A.evolve(spec, lapf, bdiag, psi0)
    torch.cuda.synchronize()
    tf = time.perf_counter() - t0
    out["splitstep_folded_steps_per_s"] = {
        "value": stepsf / tf, "unit": "steps/s", "steps": stepsf, "seconds": tf,
        "rel_diff_vs_dense": float(torch.linalg.norm(statef - state) / torch.linalg.norm(state)),
        "config": "variant of splitstep_steps_per_s: same run, A = the even/odd folded -Delta "
                  "(kronop_op_create_folded)"}
    try:  # variant: the dense kinetic operator on the INT8 path (kronop_op_set_precision)
        lap.set_precision("ozaki")
        A.evolve(A.SplitSpec(quad_points=1, dt=1e-3, total_time=5e-3, merge_across_steps=True),
                 lap, bdiag, psi0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        stateo, _, stepso = A.evolve(spec, lap, bdiag, psi0)
        torch.cuda.synchronize()
        to = time.perf_counter() - t0
        lapf.set_precision("ozaki")
        A.evolve(A.SplitSpec(quad_points=1, dt=1e-3, total_time=5e-3, merge_across_steps=True),
                 lapf, bdiag, psi0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        statefo, _, stepsfo = A.evolve(spec, lapf, bdiag, psi0)
        torch.cuda.synchronize()
        tfo = time.perf_counter() - t0
        out["splitstep_folded_ozaki_steps_per_s"] = {
            "value": stepsfo / tfo, "unit": "steps/s", "steps": stepsfo, "seconds": tfo,
            "rel_diff_vs_dense": float(torch.linalg.norm(statefo - state) / torch.linalg.norm(state)),
            "config": "variant of splitstep_steps_per_s: folded kinetic operator on the INT8 path"}
        del statefo
        out["splitstep_ozaki_steps_per_s"] = {
            "value": stepso / to, "unit": "steps/s", "steps": stepso, "seconds": to,
            "rel_diff_vs_dense": float(torch.linalg.norm(stateo - state) / torch.linalg.norm(state)),
            "config": "variant of splitstep_steps_per_s: same run, the kinetic propagate on FP64 "
                      "emulated on the INT8 tensor cores (Ozaki, 7 slices)"}
        del stateo
    except Exception as e:  # reported, never silently replaced
        out["splitstep_ozaki_steps_per_s"] = {"error": str(e)[:200]}
    del lap, lapf, bdiag, psi0, state, statef
    torch.cuda.empty_cache()
    # BASELINE configs[1] second half: exp(-i dt (-Delta+V1)) on the 1024^3 grid, complex128
    g = A.Grid.sem(8.0, 205, 5, 3)
    op = g.separable_operator(ctx, [lambda t: t * t] * 3)
    N = g.node_count()
    psi = torch.view_as_complex(A.splitmix_uniform(ctx, 7, 2 * N).view(-1, 2))
    o = torch.empty_like(psi)
    op.propagate(psi, 0.01, out=o)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(ctx.stream)
    for _ in range(2):
        op.propagate(psi, 0.01, out=o)
    e1.record(ctx.stream)
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 2e3
    out["propagate_1024"] = {
        "value": N / t / 1e9, "unit": "GDoF/s", "ms_per_step": t * 1e3,
        "tflops": 24.0 * 1024 ** 4 / t / 1e12,
        "config": "exp(-i dt (-Delta+V1)), harmonic V1, 1024^3 complex128 (BASELINE configs[1]), "
                  "dt = 0.01, phase fused into the last forward pass"}
    del op
    torch.cuda.empty_cache()
    try:  # variant: the same propagate through the even/odd folded operator
        fo = g.separable_operator(ctx, [lambda t: t * t] * 3, folded=True)
        of = torch.empty_like(psi)
        fo.propagate(psi, 0.01, out=of)
        pd = float(torch.linalg.norm(of - o) / torch.linalg.norm(o))
        torch.cuda.synchronize()
        e0.record(ctx.stream)
        for _ in range(2):
            fo.propagate(psi, 0.01, out=of)
        e1.record(ctx.stream)
        torch.cuda.synchronize()
        tfo = e0.elapsed_time(e1) / 2e3
        out["propagate_1024_folded"] = {
            "value": N / tfo / 1e9, "unit": "GDoF/s", "ms_per_step": tfo * 1e3,
            "rel_diff_vs_dense": pd,
            "config": "variant of propagate_1024: even/odd folded transforms (kronop_op_create_folded)"}
        del fo, of
    except Exception as e:  # reported, never silently replaced
        out["propagate_1024_folded"] = {"error": str(e)[:200]}
    try:  # variant: FP64 emulated on the INT8 tensor cores (Ozaki, 7 slices)
        op = g.separable_operator(ctx, [lambda t: t * t] * 3)
        oo = torch.empty_like(psi)
        op.propagate_lowp(psi, 0.01, "ozaki", out=oo)
        pd = float(torch.linalg.norm(oo - o) / torch.linalg.norm(o))
        torch.cuda.synchronize()
        e0.record(ctx.stream)
        for _ in range(2):
            op.propagate_lowp(psi, 0.01, "ozaki", out=oo)
        e1.record(ctx.stream)
        torch.cuda.synchronize()
        too = e0.elapsed_time(e1) / 2e3
        out["propagate_1024_ozaki"] = {
            "value": N / too / 1e9, "unit": "GDoF/s", "ms_per_step": too * 1e3,
            "rel_diff_vs_fp64": pd,
            "config": "variant of propagate_1024: INT8 tcgen05 products of 7 base-254 slices "
                      "(re / im as separate real rows), FP64 phase epilogue"}
        del op, oo
    except Exception as e:  # reported, never silently replaced
        out["propagate_1024_ozaki"] = {"error": str(e)[:200]}
    del psi, o
    torch.cuda.empty_cache()
    # BASELINE config 5 kernels: one complex propagate of the kinetic split (the A-step of
    # qHOP/Strang) on the 6D n = 29 and 9D n = 9 grids -- the Kronecker-factored path
    # (kron_prop.cu: (x)_a E_a, groups of 3 axes on DFMA at n = 9, of 2 on parity-folded DMMA at
    # n = 29) -- and Strang steps/s (qHOP M = 1, merged) with a B phase on the same grids.
    peaks = load_peaks()
    for name, (L_, cells, k, d) in {"6d_n29": (5.0, 3, 10, 6), "9d_n9": (3.0, 2, 5, 9)}.items():
        g = A.Grid.sem(L_, cells, k, d)
        lap = g.laplacian(ctx)
        N = g.node_count()
        psi = torch.view_as_complex(A.splitmix_uniform(ctx, 3, 2 * N).view(-1, 2))
        o = torch.empty_like(psi)
        c0 = ctx.launch_count()
        lap.propagate(psi, 0.005, out=o)
        launches = ctx.launch_count() - c0
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(ctx.stream)
        for _ in range(3):
            lap.propagate(psi, 0.005, out=o)
        e1.record(ctx.stream)
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 3e3
        n = g.shape[0]
        flops_ref = 8.0 * d * n * N  # 8 (sum n_a) N for a complex propagate
        bytes_kron = launches * 2 * 16.0 * N  # each group launch reads and writes the field
        t_fp64 = flops_ref / (peaks["fp64_tflops"] * 1e12)
        t_hbm = bytes_kron / (peaks["hbm_gbs"] * 1e9)
        rec = {
            "value": t * 1e3, "unit": "ms", "dof": N, "d": d, "n": n, "launches": launches,
            "hbm_gbs": bytes_kron / t / 1e9,
            "tflops_ref_equiv": flops_ref / t / 1e12,
            "roofline": {"bound": "fp64" if t_fp64 >= t_hbm else "hbm",
                         "fp64_bound_ms": t_fp64 * 1e3, "hbm_bound_ms": t_hbm * 1e3,
                         "frac": max(t_fp64, t_hbm) / t,
                         "note": "fp64 bound = the reference algorithm's flops (8 d n N) at the "
                                 "measured DGEMM rate; hbm bound = the launches' field round "
                                 "trips at the measured copy bandwidth",
                         "own_algorithm": own_bound(d, n, N, t, t_hbm)},
            "config": "exp(-i dt (-Delta)) on %dD SEM n=%d complex128 (BASELINE configs[4] "
                      "kinetic step), dt = 0.005, Kronecker-factored: %d group launches, no "
                      "phase pass" % (d, n, launches)}
        del o
        # Strang (qHOP M = 1, merged, dt = 0.005, T = 0.1 as in the config) with B = a separable
        # harmonic trap on the grid: per step one A propagation with the previous B phase as its
        # prologue
        try:
            b = torch.from_numpy(np.ascontiguousarray(
                P.separable_sum(g, P.build_potential("harmonic", g)))).to(device)
            A.evolve(A.SplitSpec(quad_points=1, dt=0.005, total_time=0.01, merge_across_steps=True),
                     lap, b, psi, stationary_eigenvalue=0.0)
            torch.cuda.synchronize()
            e0.record(ctx.stream)
            st, err, steps = A.evolve(A.SplitSpec(quad_points=1, dt=0.005, total_time=0.1,
                                                  merge_across_steps=True),
                                      lap, b, psi, stationary_eigenvalue=0.0)
            e1.record(ctx.stream)
            torch.cuda.synchronize()
            rec["strang_steps_per_s"] = steps / (e0.elapsed_time(e1) / 1e3)
            del st, b
        except Exception as e:  # reported, never silently replaced
            rec["strang_error"] = str(e)[:200]
        out["config5_propagate_" + name] = rec
        del lap, psi
        torch.cuda.empty_cache()
    return out


def own_bound(d, n, N, t, t_hbm):
    """Roofline of the algorithm the Kronecker propagate actually runs on the config-5 grids (the
    axes are parity-symmetric, so the folded blocks: per complex fiber and axis (M+c)^2 + M^2
    complex multiply-adds = 8 ((M+c)^2 + M^2) flops, M = n / 2), at the FP64 instruction peak of
    the unit it runs on (DFMA for n <= 10, DMMA above; profiles/r01_fp64_instr_peak.txt) against
    the same HBM bound."""
    m, me = n // 2, n // 2 + n % 2
    flops = d * (N / n) * 8.0 * (me * me + m * m)
    peak, unit = (33.92, "DFMA") if n <= 10 else (36.97, "DMMA")
    t_fp = flops / (peak * 1e12)
    return {"flops": flops, "peak_tflops": peak, "unit": unit, "fp64_bound_ms": t_fp * 1e3,
            "hbm_bound_ms": t_hbm * 1e3, "bound": "fp64" if t_fp >= t_hbm else "hbm",
            "frac": max(t_fp, t_hbm) / t}


def folded_variant(A, grid, pot, ctx, b, x, bn, xn, op_dense, steps, world, local):
    """Same 1024^3 solve through the even/odd folded operator (kronop_op_create_folded): the
    harmonic trap on the symmetric SEM grid commutes with x -> -x per axis, so every transform
    splits into two half-size blocks (half the flops, plus one fold/unfold HBM round trip per
    axis and direction). Reported beside the headline, not in it: the headline `value` and the
    roofline stay on the dense transform the reference runs."""
    import torch
    fo = grid.separable_operator(ctx, pot.separable, folded=True)
    fo.solve(b, out=x)
    ref = op_dense.solve(b)
    err = float(torch.linalg.norm(x - ref) / torch.linalg.norm(ref))
    del ref
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    k = max(1, steps)
    e0.record(ctx.stream)
    for _ in range(k):
        fo.solve(b, out=x)
    e1.record(ctx.stream)
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 1e3 / k
    t = max_over_ranks(world, t, "cuda:%d" % local)
    fo.solve_host(bn, xn)
    t0 = time.perf_counter()
    for _ in range(min(k, 3)):
        fo.solve_host(bn, xn)
    te = (time.perf_counter() - t0) / min(k, 3)
    te = max_over_ranks(world, te, "cuda:%d" % local)
    N = grid.node_count()
    fz = {}
    try:  # the folded operator on the INT8 path (kronop_op_set_precision)
        fo.set_precision("ozaki")
        fo.solve(b, out=x)
        ref = op_dense.solve(b)
        ferr = float(torch.linalg.norm(x - ref) / torch.linalg.norm(ref))
        del ref
        torch.cuda.synchronize()
        e0.record(ctx.stream)
        for _ in range(k):
            fo.solve(b, out=x)
        e1.record(ctx.stream)
        torch.cuda.synchronize()
        tz = max_over_ranks(world, e0.elapsed_time(e1) / 1e3 / k, "cuda:%d" % local)
        fz = {"folded_ozaki_solve": {
            "value": world * N / tz / 1e9, "unit": "GDoF/s", "ms_per_step": tz * 1e3,
            "rel_diff_vs_dense": ferr,
            "config": "same workload; even/odd folded transforms, each half on the INT8 path "
                      "(Ozaki, 7 slices)"}}
    except Exception as e:  # reported, never silently replaced
        fz = {"folded_ozaki_solve": {"error": str(e)[:200]}}
    del fo
    torch.cuda.empty_cache()
    # the paper's BF16 mode on the tcgen05 tensor cores: BF16 storage, FP32
    # accumulation in TMEM; separate line, accuracy ~1e-2 by construction
    bf = {}
    try:
        xb = torch.empty_like(x)
        op_dense.solve_bf16(b, out=xb)
        ref = op_dense.solve(b)
        bf_err = float(torch.linalg.norm(xb - ref) / torch.linalg.norm(ref))
        del ref
        torch.cuda.synchronize()
        e0.record(ctx.stream)
        for _ in range(k):
            op_dense.solve_bf16(b, out=xb)
        e1.record(ctx.stream)
        torch.cuda.synchronize()
        tb = max_over_ranks(world, e0.elapsed_time(e1) / 1e3 / k, "cuda:%d" % local)
        try:
            with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
                bf16_peak = json.load(f).get("bf16_tflops_sustained")
        except (OSError, ValueError):
            bf16_peak = None
        n1 = grid.shape[0]
        bf = {"bf16_solve": {
            "value": world * N / tb / 1e9, "unit": "GDoF/s", "ms_per_step": tb * 1e3,
            "rel_diff_vs_fp64": bf_err,
            "tflops": 12.0 * n1 ** 4 / tb / 1e12,
            "frac_of_bf16_peak": (12.0 * n1 ** 4 / tb / 1e12 / bf16_peak) if bf16_peak else None,
            "bf16_peak_src": "MEASURED_PEAKS.json bf16_tflops_sustained (cuBLAS)",
            "config": "same workload; BF16 storage / FP32 accumulation, tcgen05.mma kind::f16 "
                      "(M128 N256 K16) with TMEM accumulators, TMA 128B-swizzled operands; "
                      "FP64 in/out"}}
        del xb
        torch.cuda.empty_cache()
        xt = torch.empty_like(x)
        op_dense.solve_lowp(b, "tf32", out=xt)
        ref = op_dense.solve(b)
        tf_err = float(torch.linalg.norm(xt - ref) / torch.linalg.norm(ref))
        del ref
        torch.cuda.synchronize()
        e0.record(ctx.stream)
        for _ in range(k):
            op_dense.solve_lowp(b, "tf32", out=xt)
        e1.record(ctx.stream)
        torch.cuda.synchronize()
        tt = max_over_ranks(world, e0.elapsed_time(e1) / 1e3 / k, "cuda:%d" % local)
        bf["tf32_solve"] = {
            "value": world * N / tt / 1e9, "unit": "GDoF/s", "ms_per_step": tt * 1e3,
            "rel_diff_vs_fp64": tf_err,
            "config": "same workload; FP32 storage / TF32 products / FP32 accumulation, "
                      "tcgen05.mma kind::tf32 (M128 N256 K8), TMEM accumulators; FP64 in/out"}
        del xt
        torch.cuda.empty_cache()
        xf = torch.empty_like(x)
        op_dense.solve_lowp(b, "fp32", out=xf)
        ref = op_dense.solve(b)
        f3_err = float(torch.linalg.norm(xf - ref) / torch.linalg.norm(ref))
        del ref
        torch.cuda.synchronize()
        e0.record(ctx.stream)
        for _ in range(k):
            op_dense.solve_lowp(b, "fp32", out=xf)
        e1.record(ctx.stream)
        torch.cuda.synchronize()
        tf = max_over_ranks(world, e0.elapsed_time(e1) / 1e3 / k, "cuda:%d" % local)
        bf["fp32_solve"] = {
            "value": world * N / tf / 1e9, "unit": "GDoF/s", "ms_per_step": tf * 1e3,
            "rel_diff_vs_fp64": f3_err,
            "config": "same workload; FP32-level via 3xTF32: (hi, lo) TF32 pairs, three "
                      "tcgen05.mma kind::tf32 (M128 N128 K8) per term into an FP32 TMEM accumulator"}
        del xf
        torch.cuda.empty_cache()
        # FP64 emulated on the INT8 tensor cores (Ozaki scheme, 7 signed slices of base 254,
        # 28 exact INT8 products per transform): FP64-level agreement with the DMMA path
        xo = torch.empty_like(x)
        op_dense.solve_lowp(b, "ozaki", out=xo)
        ref = op_dense.solve(b)
        oz_err = float(torch.linalg.norm(xo - ref) / torch.linalg.norm(ref))
        oz_max = float((xo - ref).abs().max() / ref.abs().max())
        del ref
        torch.cuda.synchronize()
        e0.record(ctx.stream)
        for _ in range(k):
            op_dense.solve_lowp(b, "ozaki", out=xo)
        e1.record(ctx.stream)
        torch.cuda.synchronize()
        to = max_over_ranks(world, e0.elapsed_time(e1) / 1e3 / k, "cuda:%d" % local)
        int8_tops = 28 * 12.0 * n1 ** 4 / to / 1e12
        bf["ozaki_fp64_solve"] = {
            "value": world * N / to / 1e9, "unit": "GDoF/s", "ms_per_step": to * 1e3,
            "rel_diff_vs_fp64": oz_err, "max_rel_diff_vs_fp64": oz_max,
            "speedup_vs_dmma_fp64": None,
            "int8_tops": int8_tops,
            "frac_of_int8_peak": (int8_tops / (2 * bf16_peak)) if bf16_peak else None,
            "int8_peak_src": "2 x MEASURED_PEAKS.json bf16_tflops_sustained (dense INT8 = 2x BF16 "
                             "on sm_100)",
            "config": "same workload; FP64 emulation: per-row power-of-two scales, 7 signed "
                      "8-bit slices (base 254) per operand, 28 tcgen05.mma kind::i8 "
                      "(M128 N64 K32) products into 7 INT32 TMEM accumulators, FP64 Horner "
                      "combination + FP64 spectral divide in the epilogue; HBM-bound split "
                      "kernel between passes"}
        del xo
        torch.cuda.empty_cache()
    except Exception as e:  # reported, never silently replaced
        bf = {"bf16_solve": {"error": str(e)[:200]}}
    return {**bf, **fz, "folded_solve": {
        "value": world * N / t / 1e9, "unit": "GDoF/s", "ms_per_step": t * 1e3,
        "e2e": {"value": world * N / te / 1e9, "unit": "GDoF/s", "ms_per_step": te * 1e3},
        "rel_diff_vs_dense": err,
        "config": "same workload as the headline; even/odd folded transforms"}}


def run_kronop(args):
    import torch
    world, rank, local = dist_init()
    torch.cuda.set_device(local)
    from paper_2605_20491_b200 import api as A
    from paper_2605_20491_b200 import potentials as P
    peaks = load_peaks()
    n = args.n
    cells = workload_config(n)
    grid = A.Grid.sem(8.0, cells, workload_degree(n), 3)
    pot = P.build_potential("harmonic", grid)
    ctx = A.Context(local)
    op = grid.separable_operator(ctx, pot.separable)
    N = grid.node_count()
    b = A.splitmix_uniform(ctx, 1, N)
    x = torch.empty_like(b)
    stream = ctx.stream
    # warm-up (also sizes the workspace)
    for _ in range(args.warmup):
        op.solve(b, out=x)
    torch.cuda.synchronize()
    launches0 = ctx.launch_count()
    sampler = ClockSampler(local)
    barrier(world)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        op.solve(b, out=x)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    clocks = sampler.stop()
    t_step = e0.elapsed_time(e1) / 1e3 / args.steps
    launches = ctx.launch_count() - launches0
    t_step = max_over_ranks(world, t_step, "cuda:%d" % local)
    value = world * N / t_step / 1e9

    x_host = x.cpu().numpy() if (rank == 0 and not args.no_cpu) else None
    # dominant kernel: the TMA/DMMA mode-product kernel, timed pass by pass as the solve runs it
    # (forward axes 0, 1, 2 with the spectral divide fused into the axis-2 pass, backward axes
    # 0, 1, 2), CUDA events on the context stream; achieved = 2 n^4 flops per launch over the
    # mean launch time of the six
    y = torch.empty_like(b)
    seq = [(0, True, "store"), (1, True, "store"), (2, True, "div"),
           (0, False, "store"), (1, False, "store"), (2, False, "store")]
    for a_, f_, e_ in seq:
        op.transform_pass_ex(b, a_, f_, e_, out=y)
    reps = 3
    pe0 = torch.cuda.Event(enable_timing=True)
    pe1 = torch.cuda.Event(enable_timing=True)
    per_pass = []
    for a_, f_, e_ in seq:
        torch.cuda.synchronize()
        pe0.record(stream)
        for _ in range(reps):
            op.transform_pass_ex(b, a_, f_, e_, out=y)
        pe1.record(stream)
        torch.cuda.synchronize()
        per_pass.append(pe0.elapsed_time(pe1) / 1e3 / reps)
    pass_flops = 2.0 * n * N
    # the solve is exactly six launches of the pass kernel (rotated passes, the divide fused into
    # the third): its average launch duration over the timed region is t_step / 6
    launches_per_solve = launches / max(1, args.steps)
    achieved = pass_flops / (t_step / 6.0) / 1e12
    del y

    # end-to-end through the C-ABI host entry point (pinned host buffers, H2D + D2H inside)
    bh = torch.empty(N, dtype=torch.float64, pin_memory=True)
    xh = torch.empty(N, dtype=torch.float64, pin_memory=True)
    bh.copy_(b.cpu())
    bn, xn = bh.numpy(), xh.numpy()
    op.solve_host(bn, xn)  # warm (sizes the staging buffers)
    e2e_steps = max(1, min(args.steps, 5))
    barrier(world)
    e2e_ts = []
    for _ in range(e2e_steps):  # single-call latency: median step (host-memory / PCIe noise)
        t0 = time.perf_counter()
        op.solve_host(bn, xn)
        e2e_ts.append(time.perf_counter() - t0)
    t_single = float(np.median(e2e_ts))
    t_single = max_over_ranks(world, t_single, "cuda:%d" % local)
    # headline e2e: the K timed steps as one batch through kronop_sep_solve_host_batch -- every
    # step still uploads its 8 GiB right-hand side from pinned host memory and downloads its
    # 8 GiB solution, but step i+1's upload and step i-1's download run on the copy engines
    # while step i computes (a stream of solves, as a caller looping over fields issues them)
    kb = max(2, args.steps)
    op.solve_host_batch([bn, bn], [xn, xn])  # warm (sizes the batch staging)
    barrier(world)
    t0 = time.perf_counter()
    op.solve_host_batch([bn] * kb, [xn] * kb)
    t_e2e = (time.perf_counter() - t0) / kb
    t_e2e = max_over_ranks(world, t_e2e, "cuda:%d" % local)
    e2e_value = world * N / t_e2e / 1e9
    ctx.trim()  # the host-path staging (6 fields) is not needed by the measurements below

    variants = {} if args.no_extras else folded_variant(A, grid, pot, ctx, b, x, bn, xn, op,
                                                        args.steps, world, local)
    oz = variants.get("ozaki_fp64_solve")
    if oz and oz.get("ms_per_step"):
        oz["speedup_vs_dmma_fp64"] = t_step * 1e3 / oz["ms_per_step"]
    extras = {} if args.no_extras else secondary_metrics(A, P, ctx, local)
    cpu = None
    if rank == 0 and not args.no_cpu:
        cpu = cpu_leg(n, bn, x_host)
        del x_host
    if rank == 0:
        line = {
            "metric": "(-Delta+V1)^-1 apply GDoF/s at 1024^3 fp64",
            "value": value, "unit": "GDoF/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "3D (-Delta+V1)^-1 solve, harmonic V1, SEM Q%d %d cells L=8, "
                                   "n=%d (BASELINE configs[1])" % (workload_degree(n), cells, n),
                       "n": n, "dof": N, "parallelism": "replicas" if world > 1 else "single",
                       "l2": "inputs (8 GiB/field) larger than L2; no flush"},
            "tflops": 12.0 * n ** 4 / t_step / 1e12,
            "roofline": {"bound": "tensor", "achieved": achieved,
                         "peak": peaks["fp64_tflops"], "unit": "TFLOP/s",
                         "frac": achieved / peaks["fp64_tflops"],
                         "traffic": load_pass_traffic(),
                         "traffic_algorithmic": 16 * N,
                         "kernel": "mode_product_tma_kernel (TMA + FP64 DMMA), one 1024^3 pass = "
                                   "2 n^4 flops; achieved = 2 n^4 / (solve time / 6): the solve "
                                   "is six launches of it (rotated passes, divide fused into the "
                                   "third), timed over the bench's timed region",
                         "launches_per_solve": launches_per_solve,
                         "axis_order_pass_ms": [round(t * 1e3, 3) for t in per_pass],
                         "axis_order_passes": "kronop_op_pass_ex in axis order (fwd a0, a1, a2 + "
                                              "divide, bwd a0, a1, a2; STRIDED loader on axes 1-2), "
                                              "for comparison with the rotated solve",
                         "solve_frac": 12.0 * n ** 4 / t_step / 1e12 / peaks["fp64_tflops"],
                         "peak_src": peaks["fp64_src"]},
            "rel_diff_vs_oracle": cpu["rel_diff_vs_oracle"] if cpu else None,
            "e2e": {"value": e2e_value, "unit": "GDoF/s", "h2d_bytes_per_step": 8 * N,
                    "d2h_bytes_per_step": 8 * N, "ms_per_step": t_e2e * 1e3,
                    "aggregate": "%d steps as one kronop_sep_solve_host_batch call (copies of "
                                 "neighbouring steps overlapped with each step's solve), host "
                                 "wall clock / steps" % kb,
                    "single_call": {"value": world * N / t_single / 1e9, "unit": "GDoF/s",
                                    "ms_per_step": t_single * 1e3,
                                    "step_ms": [round(t * 1e3, 1) for t in e2e_ts],
                                    "aggregate": "median kronop_sep_solve_host call"}},
            "gpu_launches": int(launches),
            "secondary": extras,
            "variants": variants,
            "clocks": clocks,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


def run_kronop_slab(args):
    """N > 1 (one process per GPU, launched by torch.distributed.run): the same solve,
    slab-decomposed through the C-ABI (kronop_slab_create_nccl, csrc/slab.cu): axes 0-1 local,
    two NCCL all-to-all transposes (grouped send / recv per plane) for the last axis. Total work
    fixed => "scaling": "strong"; time = max over ranks of the CUDA-event time on the rank's
    stream. --extent 2048 runs the 2048^3 scaling grid (Q3 x 683 cells, 64 GiB per field)."""
    import torch
    import torch.distributed as dist
    world, rank, local = dist_init()
    torch.cuda.set_device(local)
    from paper_2605_20491_b200 import api as A
    from paper_2605_20491_b200 import slab as S
    peaks = load_peaks()
    n = args.n
    grid = A.Grid.sem(8.0, workload_config(n), workload_degree(n), 3)
    ax = A.build_axis(grid.axes[0], fvals=np.array([float(x) * float(x)
                                                     for x in grid.axes[0].nodes]))
    ctx = A.Context(local)
    uid = [S.nccl_unique_id() if rank == 0 else None]
    if world > 1:
        dist.broadcast_object_list(uid, src=0)
    so = S.DeviceSlabOperator([ax] * 3, ctx=ctx, rank=rank, nranks=world, unique_id=uid[0])
    pt = so.parts[0]
    plane = n * n
    b = [A.splitmix_uniform(ctx, 1, pt["elems"], start=pt["z0"] * plane)]
    x = [torch.empty_like(b[0])]
    stream = pt["stream"]
    for _ in range(args.warmup):
        so.solve(b, out=x)
    torch.cuda.synchronize()
    launches0 = ctx.launch_count()
    sampler = ClockSampler(local)
    barrier(world)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        so.solve(b, out=x)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    clocks = sampler.stop()
    t_step = max_over_ranks(world, e0.elapsed_time(e1) / 1e3 / args.steps, "cuda:%d" % local)
    launches = ctx.launch_count() - launches0
    N = n ** 3
    value = N / t_step / 1e9
    # end to end: this rank's slab from pinned host memory, solve, back to pinned host memory
    bh = torch.empty(pt["elems"], dtype=torch.float64, pin_memory=True)
    bh.copy_(b[0].cpu())
    xh = torch.empty(pt["elems"], dtype=torch.float64, pin_memory=True)
    k = max(1, min(args.steps, 3))
    barrier(world)
    t0 = time.perf_counter()
    for _ in range(k):
        bd = [bh.to("cuda:%d" % local, non_blocking=True)]
        xd = so.solve(bd)
        xh.copy_(xd[0], non_blocking=True)
        torch.cuda.synchronize()
    t_e2e = max_over_ranks(world, (time.perf_counter() - t0) / k, "cuda:%d" % local)
    tfl = 12.0 * n ** 4 / t_step / 1e12
    if rank == 0:
        line = {
            "metric": "(-Delta+V1)^-1 apply GDoF/s at 1024^3 fp64",
            "value": value, "unit": "GDoF/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "3D (-Delta+V1)^-1 solve, harmonic V1, SEM Q%d %d cells L=8, "
                                   "n=%d, slab-decomposed over %d GPUs through kronop_slab_* "
                                   "(NCCL ranks, 2 transposes per solve)"
                                   % (workload_degree(n), workload_config(n), n, world),
                       "exchange": ("fused: the pass before each transpose stores into the peers' "
                                    "CUDA-IPC-mapped slab buffers (%d solves fused)"
                                    % so.fused_transforms() if so.fused_transforms() > 0 else
                                    "NCCL grouped send / recv"),
                       "n": n, "dof": N, "parallelism": "slab%d" % world,
                       "l2": "inputs larger than L2; no flush"},
            "tflops": tfl,
            "roofline": {"bound": "tensor", "achieved": tfl / world, "peak": peaks["fp64_tflops"],
                         "unit": "TFLOP/s", "frac": tfl / world / peaks["fp64_tflops"],
                         "traffic": None, "note": "per-GPU FLOP rate of the whole slab solve "
                                                  "(transposes included)"},
            "e2e": {"value": N / t_e2e / 1e9, "unit": "GDoF/s",
                    "h2d_bytes_per_step": 8 * pt["elems"], "d2h_bytes_per_step": 8 * pt["elems"],
                    "ms_per_step": t_e2e * 1e3, "per_rank_bytes": True},
            "gpu_launches": int(launches),
            "clocks": clocks,
            "cpu_baseline": None,
        }
        print(json.dumps(line), flush=True)
    so.close()
    if dist.is_initialized():
        dist.destroy_process_group()
    return 0


def self_launch(args):
    """`bench.py --gpus N` without a launcher: re-run under torch.distributed.run with N ranks."""
    import socket
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           "--nproc-per-node", str(args.gpus), "--master-addr", "127.0.0.1", "--master-port",
           str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="kronop", choices=["kronop", "reference"])
    ap.add_argument("--extent", dest="n", type=int, default=1024,
                    help="grid extent per axis (1024 = Q5 x 205 cells; 2048 = Q3 x 683 cells)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--slab", action="store_true", help="force the slab-decomposed path (any N)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(args)
    if args.impl == "reference":
        return run_reference(args)
    if int(os.environ.get("WORLD_SIZE", "1")) > 1 or args.slab:
        return run_kronop_slab(args)
    return run_kronop(args)


if __name__ == "__main__":
    sys.exit(main())
