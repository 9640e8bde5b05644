"""configs[3] grid (the 1 mm head, 200 x 240 x 200, PWL N system, 60 components rank 25): the full
restarted GMRES(50) solve to 1e-6 on the device against the oracle's gmres (solver.hpp:34-142)
on the same forms, eps and rhs.  The oracle keeps 51 basis vectors of 1.84 GB on the host
(~125 GB with its matvec buffers) and runs ~50 full C4 matvecs (~1 h on 16 cores), so this is
a script, not a test.  argv: [inner outer tol] (default 50 200 1e-6: the full solve, ~1 h of
oracle time; "20 1 1e-14" = the first 20 Arnoldi steps, ~25 min, compared step by step).
Writes JSON lines as results arrive (the GPU part first)."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1811_00484_b200 as vie
from oracle import oracle as orc
from tests.helpers import fourier_forms, random_field, spatial_tucker_forms

orc.set_threads(os.cpu_count() or 1)
N, PWL = 0, 1
grid = (200, 240, 200)
inner, outer, tol = (int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3])) if len(sys.argv) > 3 else (50, 200, 1e-6)
nv = int(np.prod(grid))
dft = vie.DftService(0)
rng = np.random.default_rng(7)
eps_np = 1 + rng.uniform(1, 5, nv) - 1j * rng.uniform(0, 1, nv)
spatial, par = spatial_tucker_forms(N, PWL, grid, 25, 1357)
comps, _, _ = vie.component_table(N, PWL)


def build(scale):
    forms = [vie.TuckerForm(dft, grid, spatial[c][0] * scale, spatial[c][1], par[c]) for c in range(len(comps))]
    return vie.build_operator_spectra(N, PWL, grid, comps, forms, dft)


x = torch.from_numpy(random_field(PWL, grid, 1358)).cuda()
op1 = build(1.0)
rho = float(torch.linalg.vector_norm(vie.apply_operator(op1, x)) / torch.linalg.vector_norm(x))
del op1, x
torch.cuda.empty_cache()
emax = float(np.max(np.abs(eps_np - 1.0)))
gmin = float(np.min(np.abs(eps_np))) / 12.0
scale = 0.2 * gmin / (emax * rho)
op = build(scale)
rhs = random_field(PWL, grid, 17)
eps = torch.from_numpy(eps_np).cuda()
out = {"config": f"head_1mm (200, 240, 200) PWL N system, 60 components rank 25, synthetic; GMRES({inner}) x {outer} "
                 f"restarts to {tol}"}
for strategy in ("hosvd_decompress", "hosvd_loop"):
    vie.set_strategy(op, strategy)
    t0 = time.perf_counter()
    r = vie.gmres(op, eps, 1.0, torch.from_numpy(rhs).cuda(), vie.GmresConfig(tol, inner, outer))
    torch.cuda.synchronize()
    out[strategy] = {"iterations": r.iterations, "converged": r.converged,
                     "final_relative_residual": r.final_relative_residual, "seconds": time.perf_counter() - t0,
                     "history": [float(h) for h in r.residual_history]}
    if strategy == "hosvd_decompress":
        sol = r.solution.cpu().numpy()
    del r
del op, eps
torch.cuda.empty_cache()
print(json.dumps(out), flush=True)
scaled = [(core * scale, us) for core, us in spatial]
of = fourier_forms(scaled, par)
t0 = time.perf_counter()
ref = orc.gmres_system_tucker(PWL, grid, of, eps_np, 1.0, rhs, tol=tol, inner=inner, outer=outer)
out["oracle"] = {"iterations": ref.iterations, "converged": ref.converged,
                 "final_relative_residual": ref.final_relative_residual, "seconds": time.perf_counter() - t0,
                 "threads": os.cpu_count(), "history": [float(h) for h in ref.residual_history]}
hist_err = max(abs(a - b) / max(abs(b), 1e-300) for s_ in ("hosvd_decompress", "hosvd_loop")
               for a, b in zip(out[s_]["history"], out["oracle"]["history"]))
out["history_max_rel_diff"] = hist_err
out["solution_rel_l2_decompress_vs_oracle"] = float(np.linalg.norm(sol - ref.solution) / np.linalg.norm(ref.solution))
ok = hist_err <= 1e-8 and all(abs(out[s]["iterations"] - ref.iterations) <= 1 and
         abs(out[s]["final_relative_residual"] - ref.final_relative_residual) <= 1e-8
         for s in ("hosvd_decompress", "hosvd_loop")) and out["solution_rel_l2_decompress_vs_oracle"] <= 1e-8
out["parity"] = "pass" if ok else "FAIL"
print(json.dumps(out))
