"""Repeat one matvec and compare the operator's stage buffers (octant spectra Shat, the spectral
slab B after the forward passes, Bo after the pencil stage) with the first run's, bit for bit:
localises an intermittent nondeterminism to a stage.  argv: n1 n2 n3 rank reps"""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1811_00484_b200 as vie
from tests.helpers import random_field, spatial_tucker_forms

n1, n2, n3, rank, reps = (int(a) for a in sys.argv[1:6])
dims = (n1, n2, n3)
dft = vie.DftService(0)
spatial, par = spatial_tucker_forms(0, 1, dims, rank, 13 + sum(dims))
comps, _, _ = vie.component_table(0, 1)
x = torch.from_numpy(random_field(1, dims, 91)).cuda()
L = vie.lib()
try:
    RT = C.CDLL("libcudart.so.12")
except OSError:
    RT = C.CDLL("/usr/local/cuda/lib64/libcudart.so")
RT.cudaMemcpy.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int]


def buf(op, which):
    p, n = C.c_void_p(), C.c_int64()
    assert L.vie_debug_op_buffer(op.handle, which, C.byref(p), C.byref(n)) == 0
    a = np.empty(n.value, np.complex128)
    torch.cuda.synchronize()
    assert RT.cudaMemcpy(a.ctypes.data, p.value, a.nbytes, 2) == 0  # device -> host
    return a


ref = None
bad = {0: 0, 2: 0, 3: 0, "y": 0}
where = []
for rep in range(reps):
    if rep % 10 == 0:
        forms = [vie.TuckerForm(dft, dims, spatial[c][0], spatial[c][1], par[c]) for c in range(len(comps))]
        op = vie.build_operator_spectra(0, 1, dims, comps, forms, dft)
    y = vie.apply_operator(op, x, strategy="hosvd_decompress")
    torch.cuda.synchronize()
    cur = {w: buf(op, w) for w in (0, 2, 3)}
    cur["y"] = y.cpu().numpy()
    if ref is None:
        ref = cur
        continue
    for k in cur:
        d = np.nonzero(cur[k] != ref[k])[0]
        if d.size:
            bad[k] += 1
            if len(where) < 12:
                where.append((rep, k, d.size, d[:6].tolist()))
print(f"{dims} r={rank}: runs with differences per buffer {bad} of {reps - 1}")
for w in where:
    print("  rep", w[0], "buffer", w[1], "n_diff", w[2], "first idx", w[3])
