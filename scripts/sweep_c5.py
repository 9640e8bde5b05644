"""BASELINE configs[4]: Tucker tolerance x frequency sweep on a 128^3 grid -- rank, memory
and matvec throughput, every stage on the device: Green's-tensor assembly of the 6 unique
PWC N components (vie_assemble), HOSVD compression (vie_tucker_compress_device, energy
rule), operator build and the matvec (vie_matvec, CUDA events).  Mirrors the reference's
rank_sweep / compress_report (experiments.hpp:70-107, 142-183).

  python scripts/sweep_c5.py [--n 128] [--res 2e-3] > profiles/r2/c5_sweep.json
"""
import argparse
import json
import math
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=128)
    ap.add_argument("--res", type=float, default=2e-3)  # 2 mm voxels: a 25.6 cm head-sized cube
    ap.add_argument("--freqs", default="64e6,128e6,298e6,512e6")
    ap.add_argument("--tols", default="1e-4,1e-6,1e-8,1e-10")
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    import torch

    import paper_1811_00484_b200 as vie

    dft = vie.DftService(0)
    n = args.n
    dims = (n, n, n)
    grid = vie.VoxelGrid(dims, (args.res,) * 3)
    comps, par, _ = vie.component_table(vie.KIND_N, vie.PWC)
    x = torch.randn(3 * n ** 3, dtype=torch.complex128, device="cuda")
    rows = []
    for f in [float(v) for v in args.freqs.split(",")]:
        k0 = 2 * math.pi * f / 299792458.0
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        tens = vie.assemble_operator(dft, grid, k0, vie.KIND_N)
        torch.cuda.synchronize()
        t_asm = time.perf_counter() - t0
        for tol in [float(v) for v in args.tols.split(",")]:
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            forms = [vie.tucker_compress(dft, t, dims, par[c], tol) for c, (_, t) in enumerate(tens)]
            torch.cuda.synchronize()
            t_cmp = time.perf_counter() - t0
            ranks = [list(f_.ranks) for f_ in forms]
            comp_elems = sum(r[0] * r[1] * r[2] + n * (r[0] + r[1] + r[2]) for r in ranks)
            op = vie.build_operator_spectra(vie.KIND_N, vie.PWC, dims, [c for c, _ in tens], forms, dft)
            y = torch.empty_like(x)
            for _ in range(3):
                vie.apply_operator(op, x, out=y)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(args.reps):
                vie.apply_operator(op, x, out=y)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / args.reps
            rows.append({"frequency_hz": f, "tol": tol, "n": n, "res_m": args.res,
                         "max_rank": int(max(max(r) for r in ranks)), "ranks": ranks,
                         "compressed_mb": 16.0 * comp_elems / 1e6,
                         "uncompressed_mb": 16.0 * len(comps) * n ** 3 / 1e6,
                         "compression_factor": len(comps) * n ** 3 / comp_elems,
                         "matvec_ms": ms, "matvecs_per_s": 1000.0 / ms,
                         "assembly_s": t_asm, "compress_s": t_cmp})
            print(json.dumps(rows[-1]), file=sys.stderr, flush=True)
            del op, forms
    print(json.dumps({"config": f"C5 sweep: {n}^3 PWC N, {args.res * 1e3:.1f} mm voxels, device assembly + HOSVD "
                                f"(energy rule) + matvec", "rows": rows}))


if __name__ == "__main__":
    main()
