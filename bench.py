#!/usr/bin/env python3
"""Benchmark: Tucker-compressed VIE matvecs/s at the 1 mm head grid (BASELINE.json).

One step = one apply_operator (vie_matvec) of the PWL N operator (60 unique
Tucker components, rank 25, 12 current components) on the 200 x 240 x 200 grid
(embedded 400 x 480 x 400) with synthetic spatial-domain Tucker forms
 and a synthetic current; inputs (1.84 GB) exceed the 126 MB L2.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Under torchrun (N > 1) the matvec is slab-decomposed (rank r: z-planes and
axis-2 spectral rows, two NCCL all-to-alls per matvec; component sharding with
an NCCL all-reduce when the grid does not split evenly); the time is the max
over ranks (strong scaling: the grid is fixed).  --impl reference times the CPU oracle (restatement of the
reference, which cannot be compiled here) on a bounded sample.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (grid, basis, rank)
    "head_1mm": ((200, 240, 200), 1, 25),     # BASELINE configs[3] (headline)
    "head_2mm": ((100, 120, 100), 1, 25),     # configs[2]
    "cube_64": ((64, 64, 64), 1, 25),         # configs[1]
    "cube_32": ((32, 32, 32), 1, 25),         # configs[0]
    "head_1mm_pwc": ((200, 240, 200), 0, 25),
    "cube_128": ((128, 128, 128), 1, 25),     # configs[4] grid (the C5 sweep itself: scripts/sweep_c5.py)
    "duke_head": ((93, 119, 125), 1, 25),     # the paper's Duke head grid (m = 186 = 6x31, 238 = 14x17, 250)
}
METRIC = "compressed-VIE matvecs/s at 1mm head grid; achieved HBM GB/s vs B200 peak"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="head_1mm", choices=sorted(CONFIGS))
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-solve", action="store_true")
    ap.add_argument("--slab", action="store_true", help="slab-decomposed path even on 1 GPU (exercise it)")
    ap.add_argument("--torch-exchange", action="store_true",
                    help="N > 1: exchange through torch all_to_all_single instead of the library's NCCL calls")
    ap.add_argument("--strategy", default="hosvd_decompress", choices=["hosvd_decompress", "hosvd_loop"],
                    help="MatvecStrategy of the headline (operator.hpp:17); the other one is timed beside it")
    return ap.parse_args()


def bytes_model(grid, basis, nc):
    """Algorithmic HBM bytes; B = 16 bytes per complex."""
    n1, n2, n3 = grid
    nv = n1 * n2 * n3
    ne = 8 * nv
    S = 3 if basis == 0 else 12
    noct = (n1 + 1) * (n2 + 1) * (n3 + 1)
    return {
        "matvec_staged": 16 * (2 * S) * (nv + 2 * ne),  # SURVEY bytes_mv
        # per kernel of this implementation (read + write of its operands)
        "row_fwd": 16 * S * (nv + 2 * nv),
        "col_fwd": 16 * S * (2 * nv + 4 * nv),
        "decomp": 16 * nc * noct,  # octant spectra written (Z and forms negligible)
        "pencil": 16 * (2 * S) * 4 * nv + 16 * nc * noct,  # x^/y^ slabs + octant spectra read once
        "col_inv": 16 * S * (4 * nv + 2 * nv),
        "row_inv": 16 * S * (2 * nv + nv),
    }


STAGES = ["row_fwd", "col_fwd", "decomp", "pencil", "col_inv", "row_inv"]


def flops_model(grid, basis, nc, rank):
    """Algorithmic FP64 flops.  Complex MAC = 8 flops; a length-N complex FFT is
    credited the conventional 5 N log2 N (pad/crop pruning not credited)."""
    n1, n2, n3 = grid
    m1, m2, m3 = 2 * n1, 2 * n2, 2 * n3
    S = 3 if basis == 0 else 12
    noct = (n1 + 1) * (n2 + 1) * (n3 + 1)
    nb = 9 if basis == 0 else 144
    ne = 8 * n1 * n2 * n3
    fft = lambda lines, n: 5.0 * lines * n * math.log2(n)
    return {
        "decomp": 8.0 * nc * rank * noct + 8.0 * nc * rank * rank * (n1 + 1) * (n2 + 1),
        "hadamard": 8.0 * nb * ne,
        # per kernel
        "row_fwd": fft(S * n2 * n3, m1), "col_fwd": fft(S * m1 * n3, m2),
        "pencil": 8.0 * nb * ne + 2 * fft(S * m1 * m2, m3),
        "col_inv": fft(S * m1 * n3, m2), "row_inv": fft(S * n2 * n3, m1),
    }


FP64_PEAK_TFLOPS = 37.1  # measured DMMA m8n8k4 = DFMA peak on this pool (profiles/r1_fp64_peak.txt)


# ----------------------------------------------------------------------- clocks
class ClockSampler:
    def __init__(self, gpu_index=0):
        self.samples = []
        self.proc = None
        self.gpu_index = gpu_index

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu_index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = [s for s in self.samples if len(s) >= 8]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ------------------------------------------------------------------ CPU sample
def config_dict(args, grid, basis, r, nc, S):
    """The workload description both arms print (identical dicts)."""
    return {"workload": f"{args.config}: PWL N-operator apply_operator (vie_matvec), grid {tuple(grid)}, "
                        f"embedded {tuple(2 * d for d in grid)}, {nc} Tucker components rank {r}, {S} currents",
            "grid": list(grid), "basis": "PWL" if basis else "PWC", "rank": r, "components": nc,
            "l2": "inputs 1.8 GB > 126 MB L2 (no flush needed)"}


def oracle_staged(grid, basis, rank, seed=1234):
    """The oracle's apply_operator_tucker (restated HosvdDecompress path, operator.hpp:273-382)
    as the 2S + NC pieces of ONE matvec on the bench's synthetic forms and a CN(0,1) x."""
    from oracle import oracle as orc
    from tests.helpers import fourier_forms, spatial_tucker_forms

    spatial, par = spatial_tucker_forms(0, basis, grid, rank, seed)
    forms = fourier_forms(spatial, par)
    S = 3 if basis == 0 else 12
    nv = int(np.prod(grid))
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(S * nv) + 1j * rng.standard_normal(S * nv)
    return orc.StagedMatvec(0, basis, grid, forms, x), forms


def cpu_sample(grid, basis, rank, threads, seed=1234, reps=3):
    """Bounded sample (~10-30 s) of the oracle matvec for the b200 arm's cpu_baseline:
    three real pieces of one staged C4 matvec -- forward3 of current 0, component 0's
    decompress + mac, inverse3 of target 0 -- timed (median of `reps`) and scaled to the
    matvec's 2S FFT pieces + NC component pieces.  The reference arm (--impl reference)
    times every piece of a full matvec instead."""
    from oracle import oracle as orc

    orc.set_threads(threads)
    S = 3 if basis == 0 else 12
    mv, _forms = oracle_staged(grid, basis, rank, seed)
    nc = mv.npieces - 2 * S
    t_f, t_c, t_i = [], [], []
    for _ in range(reps):
        for piece, acc in ((0, t_f), (S, t_c), (S + nc, t_i)):
            t0 = time.perf_counter()
            mv.piece(piece)
            acc.append(time.perf_counter() - t0)
    mv.close()
    tf, tc, ti = (float(np.median(v)) for v in (t_f, t_c, t_i))
    per_mv = S * tf + nc * tc + S * ti
    info = {"t_forward3_s": round(tf, 3), "t_component_s": round(tc, 3), "t_inverse3_s": round(ti, 3),
            "scaled_matvec_s": round(per_mv, 2),
            "sample": f"3 pieces of one staged oracle matvec at {tuple(grid)} (forward3 of current 0, component 0 "
                      f"decompress+mac, inverse3 of target 0; median of {reps}), scaled to {S}+{S} FFT pieces + {nc} "
                      f"component pieces; --impl reference times all pieces of a full matvec"}
    return 1.0 / per_mv, info


# ------------------------------------------------------------------ reference arm
def run_reference(args):
    """The reference's CPU path, timed on ONE full matvec: the oracle's staged
    apply_operator_tucker (all 2S + NC pieces, all host threads) spread over the K timed
    steps -- step k runs pieces [k P / K, (k + 1) P / K) of the same matvec (K > P: more
    matvecs), so the steps sum to complete matvecs and value = matvecs / total time.
    Warm-up steps run pieces of a throwaway matvec.  Plus a bounded single-thread sample
    (the reference itself is single-threaded: FFTW_ESTIMATE without threads, Eigen without
    OpenMP, proj/CMakeLists.txt:28)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import oracle as orc

    grid, basis, r = CONFIGS[args.config]
    S = 3 if basis == 0 else 12
    threads = os.cpu_count() or 1
    orc.set_threads(threads)
    t_setup = time.perf_counter()
    mv, forms = oracle_staged(grid, basis, r)
    P = mv.npieces
    nc = P - 2 * S
    t_setup = time.perf_counter() - t_setup
    for i in range(min(args.warmup, P)):  # warm-up: pieces of a throwaway matvec
        mv.piece(i)
    mv.close()
    K = max(1, args.steps)
    n_mv = max(1, -(-K // P))
    T = n_mv * P
    step_s = []
    done = 0
    for k in range(K):
        lo, hi = k * T // K, (k + 1) * T // K
        t0 = time.perf_counter()
        for i in range(lo, hi):
            j = i % P
            if j == 0:
                if done:
                    mv.close()
                mv, forms = oracle_staged(grid, basis, r, seed=1234 + done)
                done += 1
            mv.piece(j)
        step_s.append(time.perf_counter() - t0)
    mv.close()
    total = float(sum(step_s))
    val = n_mv / total
    # single-thread sample: forward3 of current 0 + component 0 (bounded, ~tens of s)
    orc.set_threads(1)
    mv1, _f = oracle_staged(grid, basis, r)
    t0 = time.perf_counter()
    mv1.piece(0)
    t_f1 = time.perf_counter() - t0
    t0 = time.perf_counter()
    mv1.piece(S)
    t_c1 = time.perf_counter() - t0
    mv1.close()
    orc.set_threads(threads)
    st_val = 1.0 / (2 * S * t_f1 + nc * t_c1)
    nv = int(np.prod(grid))
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "matvecs/s", "n_gpus": args.gpus,
        "steps": K, "warmup": args.warmup, "ms_per_step": 1000.0 * total / K, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": config_dict(args, grid, basis, r, nc, S),
        "cpu_baseline": {"value": val, "unit": "matvecs/s", "cores": threads, "kind": "port",
                         "sample": f"{n_mv} full oracle matvec(s) at {tuple(grid)} ({P} pieces: {S} forward3, {nc} "
                                   f"component decompress+mac, {S} inverse3) spread over the {K} timed steps, "
                                   f"{threads} threads"},
        "e2e": {"value": val, "unit": "matvecs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "detail": {"matvec_s": total / n_mv, "step_s": [round(t, 3) for t in step_s], "pieces_per_matvec": P,
                   "setup_s": round(t_setup, 2), "x_elems": S * nv,
                   "single_thread": {"value": st_val, "unit": "matvecs/s", "cores": 1,
                                     "sample": "forward3 of current 0 + component 0 (decompress+mac), 1 thread, "
                                               f"scaled to {2 * S} FFT + {nc} component pieces",
                                     "t_fft3_s": round(t_f1, 2), "t_component_s": round(t_c1, 2)}},
    }
    emit(line)
    return 0


# ------------------------------------------------------------------ solve time
def gmres_solve_bench(vie, dft, torch, with_cpu=True, tol=1e-6, inner=50, outer=200, grid=(64, 64, 64), reps=3):
    """Solve time (north star: matvecs/s AND solve time): restarted GMRES(50) to 1e-6 on
    the PWL system at 64^3 (BASELINE configs[1]) or the headline grid, device resident
    (vie_gmres_solve).  Synthetic rank-25 forms are scaled so |(eps - 1) N| ~ 0.2
    min|eps g| (a well-posed perturbation of the PWL Gram term); eps = 1 + U(1,5) - i U(0,1)."""
    from tests.helpers import spatial_tucker_forms

    basis, r = 1, 25
    S = vie.ncur(basis)
    nv = int(np.prod(grid))
    comps, _, _ = vie.component_table(0, basis)
    spatial, par = spatial_tucker_forms(0, basis, grid, r, 4321)

    def build(scale):
        forms = [vie.TuckerForm(dft, grid, spatial[c][0] * scale, spatial[c][1], par[c]) for c in range(len(comps))]
        return vie.build_operator_spectra(0, basis, grid, comps, forms, dft), forms

    g = torch.Generator(device="cuda").manual_seed(11)
    x = torch.randn(S * nv, dtype=torch.complex128, device="cuda", generator=g)
    op1, _ = build(1.0)
    rho = float(torch.linalg.vector_norm(vie.apply_operator(op1, x)) / torch.linalg.vector_norm(x))
    del op1
    scale = 0.2 * (2.0 / 12.0) / (5.0 * max(rho, 1e-300))  # max|eps - 1| = 5, min|eps g| = 2/12
    op, forms = build(scale)
    rng = np.random.default_rng(5)
    eps = torch.from_numpy(1 + rng.uniform(1, 5, nv) - 1j * rng.uniform(0, 1, nv)).cuda()
    rhs = torch.randn(S * nv, dtype=torch.complex128, device="cuda", generator=g)
    cfg = vie.GmresConfig(tol, inner, outer)
    vie.gmres(op, eps, 1.0, rhs, vie.GmresConfig(tol, 2, 1))  # warm-up
    times = []
    for _ in range(reps):  # min of the solves: the per-iteration host round trip sees host noise
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = vie.gmres(op, eps, 1.0, rhs, cfg)
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
    t = min(times)
    out = {"config": f"{grid} PWL N system, 60 components rank 25, synthetic",
           "solver": f"restarted GMRES({inner}) to {tol}, device resident (vie_gmres_solve)",
           "iterations": res.iterations, "converged": res.converged,
           "final_relative_residual": res.final_relative_residual, "seconds": t,
           "seconds_all": times,
           "ms_per_iteration": 1e3 * t / max(res.iterations, 1)}
    if with_cpu:  # the oracle's GMRES on the same system, bounded: 2 iterations, per-iteration time
        from oracle import oracle as orc
        from tests.helpers import fourier_forms

        scaled = [(core * scale, us) for core, us in spatial]
        of = fourier_forms(scaled, par)
        orc.set_threads(os.cpu_count() or 1)
        t0 = time.perf_counter()
        ref = orc.gmres_system_tucker(basis, grid, of, eps.cpu().numpy(), 1.0, rhs.cpu().numpy(), tol=tol,
                                      inner=2, outer=1)
        tc = (time.perf_counter() - t0) / max(ref.iterations, 1)
        out["cpu_oracle_ms_per_iteration"] = 1e3 * tc
        out["cpu_oracle_cores"] = os.cpu_count() or 1
        out["cpu_oracle_solve_seconds_estimate"] = tc * res.iterations
    return out


def gmres_solve_slab(vie, dft, torch, comm, rank, world, grid, dist, tol=1e-6, inner=50, outer=200):
    """The same solve as gmres_solve_bench at `grid`, distributed over the slab ranks: every
    vector is the rank's z-slab, each matvec is vie_slab_matvec (library exchange) and every
    dot / norm is all-reduced over `comm` (vie_gmres_solve on a partitioned operator).  Time =
    max over ranks."""
    from paper_1811_00484_b200.sharding import SlabMatvec, local_slab
    from tests.helpers import spatial_tucker_forms

    basis, r = 1, 25
    S = vie.ncur(basis)
    n1, n2, n3 = grid
    nv = int(np.prod(grid))
    comps, _, _ = vie.component_table(0, basis)
    spatial, par = spatial_tucker_forms(0, basis, grid, r, 4321)

    def build(scale):
        forms = [vie.TuckerForm(dft, grid, spatial[c][0] * scale, spatial[c][1], par[c]) for c in range(len(comps))]
        op = vie.build_operator_spectra(0, basis, grid, comps, forms, dft)
        return op, SlabMatvec(op, rank, world, comm=comm)

    def gsum(v):
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        if dist is not None:
            dist.all_reduce(t)
        return float(t.item())

    g = torch.Generator(device="cuda").manual_seed(11)
    x = local_slab(torch.randn(S * nv, dtype=torch.complex128, device="cuda", generator=g), S, n3, n1 * n2, rank,
                   world).contiguous()
    op1, sm1 = build(1.0)
    ax = sm1.apply(x)
    rho = (gsum(float(torch.linalg.vector_norm(ax)) ** 2) / gsum(float(torch.linalg.vector_norm(x)) ** 2)) ** 0.5
    del op1, sm1, ax
    scale = 0.2 * (2.0 / 12.0) / (5.0 * max(rho, 1e-300))
    op, sm = build(scale)
    rng = np.random.default_rng(5)
    eps = local_slab(torch.from_numpy(1 + rng.uniform(1, 5, nv) - 1j * rng.uniform(0, 1, nv)).cuda(), 1, n3, n1 * n2,
                     rank, world).contiguous()
    rhs = local_slab(torch.randn(S * nv, dtype=torch.complex128, device="cuda", generator=g), S, n3, n1 * n2, rank,
                     world).contiguous()
    vie.gmres(op, eps, 1.0, rhs, vie.GmresConfig(tol, 2, 1))  # warm-up
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    t0 = time.perf_counter()
    res = vie.gmres(op, eps, 1.0, rhs, vie.GmresConfig(tol, inner, outer))
    torch.cuda.synchronize()
    t = time.perf_counter() - t0
    tt = torch.tensor([t], dtype=torch.float64, device="cuda")
    if dist is not None:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t = float(tt.item())
    return {"config": f"{grid} PWL N system, 60 components rank 25, synthetic, z-slabs over {world} GPU(s)",
            "solver": f"restarted GMRES({inner}) to {tol}, distributed (vie_gmres_solve on the partitioned "
                      "operator: vie_slab_matvec + NCCL all-reduced dots)",
            "iterations": res.iterations, "converged": res.converged,
            "final_relative_residual": res.final_relative_residual, "seconds": t,
            "ms_per_iteration": 1e3 * t / max(res.iterations, 1)}


def scene_stages_bench(vie, torch, grid, peak, reps=5):
    """The solve_scene stages around the solve (build_rhs, recover_fields' e pass,
    postprocess with h; kernels_scene.cu) at the workload grid: one streaming pass
    each, so each is reported against the HBM roofline with its algorithmic bytes
    per voxel (eps 16 B, a PWC field 48 B, h_x/h_y 32 B, p_abs / b1 8 B each)."""
    n1, n2, n3 = grid
    nv = n1 * n2 * n3
    eps = torch.ones((n3, n2, n1), dtype=torch.complex128, device="cuda")
    eps[1:-1, 1:-1, 1:-1] = complex(50.0, -0.7 / (8.8541878128e-12 * 2 * np.pi * 2.98e8))
    m = vie.DielectricMap(vie.VoxelGrid(grid, (1e-3,) * 3), eps.reshape(-1), 2.98e8)
    inc = vie.PlaneWave((1, 0, 0), (0, 0, 1), 1.0)
    g = torch.Generator(device="cuda").manual_seed(3)
    j = torch.randn(3 * nv, dtype=torch.complex128, device="cuda", generator=g)
    h = torch.randn(3 * nv, dtype=torch.complex128, device="cuda", generator=g)
    f = vie.Fields(j, h, True)
    stages = {"build_rhs": (lambda: vie.build_rhs(m, inc), 16 + 48),
              "recover_e": (lambda: vie.recover_fields(j, m, inc), 16 + 48 + 48),
              "postprocess": (lambda: vie.postprocess(f, m), 16 + 48 + 32 + 8 + 8)}
    out = {"grid": list(grid), "voxels": nv}
    for name, (fn, bpv) in stages.items():
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        gbs = bpv * nv / (ms * 1e-3) / 1e9
        out[name] = {"ms": ms, "bytes_per_voxel": bpv, "achieved_gbs": gbs, "frac": gbs / peak}
    return out


# ------------------------------------------------------------------ B200 arm
def run_b200(args):
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import __graft_entry__

    __graft_entry__.build()
    import paper_1811_00484_b200 as vie
    from tests.helpers import spatial_tucker_forms

    grid, basis, r = CONFIGS[args.config]
    S = vie.ncur(basis)
    nv = int(np.prod(grid))
    n = S * nv
    comps, _, _ = vie.component_table(0, basis)
    nc = len(comps)
    # N > 1: slab decomposition (z-planes / axis-2 spectral rows, two NCCL all-to-alls per
    # matvec) when the grid splits evenly, else component sharding + NCCL all-reduce
    group = 2 * (1 if S >= 12 else (2 if S >= 6 else 4))  # axis-1 positions per pencil group
    slab = ((world > 1 or args.slab) and grid[2] % world == 0 and (2 * grid[0]) % world == 0
            and ((2 * grid[0]) // world) % group == 0)
    mine = list(range(nc)) if (world == 1 or slab) else [c for c in range(nc) if c % world == rank]
    dft = vie.DftService(local)
    spatial, par = spatial_tucker_forms(0, basis, grid, r, 1234)
    forms = [vie.TuckerForm(dft, grid, spatial[c][0], spatial[c][1], par[c]) for c in mine]
    op = vie.build_operator_spectra(0, basis, grid, [comps[c] for c in mine], forms, dft)
    g = torch.Generator(device="cuda").manual_seed(2024)
    stream = torch.cuda.Stream()  # dedicated stream: events and kernels on the same queue
    torch.cuda.set_stream(stream)
    if slab:
        from paper_1811_00484_b200.sharding import SlabMatvec, make_comm

        # the library's NCCL exchange (vie_slab_matvec: grouped send/recv, decomposition on a
        # side stream during the forward exchange); --torch-exchange: the Python stages +
        # torch all_to_all_single
        comm = None if args.torch_exchange else make_comm(dft, rank, world)
        sm = SlabMatvec(op, rank, world, comm=comm)
        x = torch.randn(sm.x_elems, dtype=torch.complex128, device="cuda", generator=g)  # this rank's z-slab
    else:
        x = torch.randn(n, dtype=torch.complex128, device="cuda", generator=g)
    y = torch.empty_like(x)

    if not slab:
        vie.set_strategy(op, args.strategy)

    def step():
        if slab:
            sm.apply(x, out=y)
            return
        vie.apply_operator(op, x, out=y, stream=stream.cuda_stream)
        if dist is not None:
            dist.all_reduce(y)

    exchange_note = None
    if slab and not args.torch_exchange:
        try:  # the first library-path matvec; a failure is recorded and the torch exchange takes over
            step()
            torch.cuda.synchronize()
        except Exception as e:  # noqa: BLE001
            exchange_note = f"library exchange failed ({type(e).__name__}: {e}); torch all_to_all_single used"
            sm = SlabMatvec(op, rank, world, comm=None)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / args.steps
    if dist is not None:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    value = 1000.0 / ms  # matvecs/s (one matvec per step for the whole job)

    # per-kernel device times over a profiled pass (CUDA events on the op stream);
    # a slab-partitioned rank profiles one unpartitioned operator of its own instead
    prof_op = op
    if slab:
        prof_op = vie.build_operator_spectra(0, basis, grid, comps, forms, dft)
        x_full = torch.randn(n, dtype=torch.complex128, device="cuda", generator=g)
    prof_x = x_full if slab else x
    prof_y = torch.empty_like(prof_x)
    prof_op.set_profiling(True)
    stage_ms = np.zeros(6)
    nprof = max(3, min(args.steps, 10))
    for _ in range(nprof):
        vie.apply_operator(prof_op, prof_x, out=prof_y, stream=stream.cuda_stream)
        launches, st = prof_op.last_stats()
        stage_ms += np.array(st[:6])
    stage_ms /= nprof
    prof_op.set_profiling(False)
    if slab:
        del prof_op, prof_x, prof_y, x_full
        launches += 1 if rank == 0 else 0  # rank 0 also decompresses octant row n2 (second launch)
    bm = bytes_model(grid, basis, len(mine))
    peak, peak_kind = measured_peak()
    dom = STAGES[int(np.argmax(stage_ms))]
    achieved = bm[dom] / (stage_ms[STAGES.index(dom)] * 1e-3) / 1e9
    traffic = None
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tf):
        try:
            traffic = json.load(open(tf)).get(args.config, {}).get(dom)
        except Exception:
            traffic = None

    # end-to-end through the reference-facing C-ABI calls with pinned host buffers:
    # every step = H2D of its x + matvec + D2H of its y.  Headline: the pipelined batch
    # call (vie_matvec_host_batch: copies of neighbouring steps overlap the matvec);
    # also reported: one synchronous vie_matvec_host call per step.
    e2e = None
    if not args.no_e2e and world == 1:
        L = vie.lib()
        xh = [torch.empty(n, dtype=torch.complex128).pin_memory() for _ in range(2)]
        yh = [torch.empty(n, dtype=torch.complex128).pin_memory() for _ in range(2)]
        xc = x.cpu()
        for t in xh:
            t.copy_(xc)
        ne2e = max(3, args.steps)

        def batch(k):
            xp = (C.c_void_p * k)(*[xh[i % 2].data_ptr() for i in range(k)])
            yp = (C.c_void_p * k)(*[yh[i % 2].data_ptr() for i in range(k)])
            assert L.vie_matvec_host_batch(op.handle, k, xp, yp) == 0

        batch(2)
        t0 = time.perf_counter()
        batch(ne2e)
        t_batch = (time.perf_counter() - t0) / ne2e
        for _ in range(2):
            assert L.vie_matvec_host(op.handle, xh[0].data_ptr(), yh[0].data_ptr()) == 0
        ns = max(2, min(args.steps, 5))
        t0 = time.perf_counter()
        for _ in range(ns):
            assert L.vie_matvec_host(op.handle, xh[0].data_ptr(), yh[0].data_ptr()) == 0
        t_sync = (time.perf_counter() - t0) / ns
        e2e = {"value": 1.0 / t_batch, "unit": "matvecs/s", "h2d_bytes_per_step": 16 * n,
               "d2h_bytes_per_step": 16 * n, "steps": ne2e,
               "api": "vie_matvec_host_batch (pinned host x_i -> y_i, copies overlapped with neighbouring matvecs)",
               "sync_call_value": 1.0 / t_sync, "sync_call_api": "vie_matvec_host (H2D, matvec, D2H serialised)"}

    # N > 1 (slab-decomposed): every rank copies its z-slab of x from pinned host memory, runs the
    # library's slab matvec (vie_slab_matvec: NCCL exchanges inside) and copies its slab of y back;
    # per-step bytes are the whole job's (all ranks' slabs); time = max over ranks
    if not args.no_e2e and slab and e2e is None:
        xh = torch.empty(sm.x_elems, dtype=torch.complex128).pin_memory()
        yh = torch.empty(sm.x_elems, dtype=torch.complex128).pin_memory()
        xh.copy_(x.cpu())
        xd, yd = torch.empty_like(x), torch.empty_like(x)

        def e2e_step():
            xd.copy_(xh, non_blocking=True)
            sm.apply(xd, out=yd)
            yh.copy_(yd, non_blocking=True)

        for _ in range(2):
            e2e_step()
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        ne2e = max(3, args.steps)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(ne2e):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        t_e = e0.elapsed_time(e1) / ne2e
        if dist is not None:
            tt = torch.tensor([t_e], device="cuda", dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t_e = float(tt.item())
        tot = 16 * sm.x_elems * world
        e2e = {"value": 1000.0 / t_e, "unit": "matvecs/s", "h2d_bytes_per_step": tot, "d2h_bytes_per_step": tot,
               "steps": ne2e, "api": f"per rank: pinned host z-slab -> device, SlabMatvec.apply (vie_slab_matvec), "
                                     f"device -> pinned host; {world} rank(s), time = max over ranks"}

    # the other MatvecStrategy on the same operator and input (operator.hpp:17-31): hosvd_decompress
    # keeps every component's octant spectrum in one HBM buffer; hosvd_loop decompresses tiles
    # into an L2-resident ring inside one persistent kernel (no whole-spectrum buffer)
    strategies = None
    if world == 1 and not slab:
        strategies = {}
        y_head = y.clone()
        n1, n2, n3 = grid
        rs = 16 * nc * (n3 + 1)
        la = int(os.environ.get("VIE_FUSED_LA", "4"))
        storage = {"hosvd_decompress": (n1 + 1) * (n2 + 1) * rs,
                   "hosvd_loop": ((la + 1) * 32 + 2 * (n1 + 1) + 2 * (n2 - 1)) * rs}
        for strat in ("hosvd_decompress", "hosvd_loop"):
            entry = {"spectrum_storage_bytes": storage[strat]}
            try:
                vie.set_strategy(op, strat)
            except ValueError as e:
                entry["unavailable"] = str(e)
                strategies[strat] = entry
                continue
            for _ in range(2):
                step()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(args.steps):
                step()
            e1.record(stream)
            torch.cuda.synchronize()
            ms_s = e0.elapsed_time(e1) / args.steps
            entry.update({"ms_per_step": ms_s, "value": 1000.0 / ms_s, "unit": "matvecs/s",
                          "rel_l2_vs_headline": float(torch.linalg.vector_norm(y - y_head)
                                                      / torch.linalg.vector_norm(y_head))})
            strategies[strat] = entry
        vie.set_strategy(op, args.strategy)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        v, info = cpu_sample(grid, basis, r, threads)
        cpu = {"value": v, "unit": "matvecs/s", "cores": threads, "kind": "port", "sample": info["sample"],
               "detail": info}

    solve = solve_c4 = None
    if rank == 0 and world == 1 and not args.no_solve:
        solve = gmres_solve_bench(vie, dft, torch, with_cpu=not args.no_cpu_baseline)
        if args.config == "head_1mm":  # the user-visible end-to-end number at the headline grid
            del op, x, y
            if e2e is not None:
                del xh, yh
            torch.cuda.synchronize()
            torch.cuda.empty_cache()
            solve_c4 = gmres_solve_bench(vie, dft, torch, with_cpu=False, grid=grid, reps=1)
    solve_dist = None
    if slab and not args.no_solve and sm.comm is not None:  # the headline solve with distributed vectors
        x = y = None  # noqa: F841  (free the matvec vectors)
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        solve_dist = gmres_solve_slab(vie, dft, torch, sm.comm, rank, world, grid, dist)
    scene = None
    if rank == 0 and world == 1 and not args.no_solve:
        scene = scene_stages_bench(vie, torch, grid, peak)

    fl = flops_model(grid, basis, nc, r)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "matvecs/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "c128",
            "data": "synthetic (spatial-domain Tucker forms, CN(0,1), parity rows zeroed; CN(0,1) currents)",
            "config": config_dict(args, grid, basis, r, nc, S),
            "parallelism": (f"slab decomposition x{world} (z-planes / axis-1 positions, NCCL all-to-all "
                            f"{'via torch' if args.torch_exchange or exchange_note else 'inside libvie_b200 (vie_slab_matvec)'})"
                            + (f"; {exchange_note}" if exchange_note else "") if slab
                            else f"components sharded x{world}") if world > 1 else "1 GPU",
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                         "algorithmic_bytes_per_launch": bm[dom]},
            "staged_model": {"bytes_per_matvec": bm["matvec_staged"],
                             "achieved_gbs": bm["matvec_staged"] / (ms * 1e-3) / 1e9,
                             "frac": bm["matvec_staged"] / (ms * 1e-3) / 1e9 / peak},
            "stage_ms": {k: round(float(v), 4) for k, v in zip(STAGES, stage_ms)},
            "fp64_gflop": {k: v / 1e9 for k, v in fl.items()},
            # the pencil kernel is FP64-pipe bound (168 GFLOP vs 24 GB at C4): the FP64 roofline
            "roofline_fp64": {"bound": "fp64", "kernel": dom, "achieved": fl[dom] / (stage_ms[STAGES.index(dom)] * 1e-3) / 1e12,
                              "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                              "frac": fl[dom] / (stage_ms[STAGES.index(dom)] * 1e-3) / 1e12 / FP64_PEAK_TFLOPS,
                              "per_kernel_tflops": {k: fl[k] / (stage_ms[STAGES.index(k)] * 1e-3) / 1e12
                                                    for k in STAGES if k in fl},
                              "peak_kind": "measured (scripts/fp64_peak.cu)"},
            "gpu_launches": launches * args.steps,
            "clocks": clk.summary(),
            "e2e": e2e,
            "strategy": args.strategy,
            "strategies": strategies,
            "cpu_baseline": cpu,
            "gmres_solve": solve,
            "gmres_solve_headline": solve_c4,
            "gmres_solve_distributed": solve_dist,
            "scene_stages": scene,
        }
        emit(line)
    if dist is not None:
        dist.destroy_process_group()
    return 0


_JSON_FD = None


def emit(line):
    """The one JSON line of the run, on the original stdout (every other byte -- NCCL banners,
    library prints -- goes to stderr, see main())."""
    data = (json.dumps(line) + "\n").encode()
    if _JSON_FD is None:
        sys.stdout.write(data.decode())
        sys.stdout.flush()
    else:
        os.write(_JSON_FD, data)


def main():
    global _JSON_FD
    # keep stdout for the JSON line alone: native code (NCCL's version banner, ...) may print on
    # file descriptor 1, so fd 1 is pointed at stderr for the rest of the run
    sys.stdout.flush()
    _JSON_FD = os.dup(1)
    os.dup2(2, 1)
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
