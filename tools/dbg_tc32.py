import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2103_01691_b200 as km
from oracle import kronmode_oracle as orc
rng = np.random.default_rng(0)
shape = (128, 128, 4)
u = np.asfortranarray((rng.standard_normal(shape) + 1j*rng.standard_normal(shape)).astype(np.complex64))
for name, mat in [("eye", np.eye(128, dtype=np.complex64)), ("rand", (rng.standard_normal((128,128))/11).astype(np.complex64))]:
    got = km.mu_mode_product(u, mat, 2)
    want = orc.mu_mode_product(u, mat, 2)
    print(name, "rel", orc.rel_l2(got, want), "max|got|", np.abs(got).max(), "max|want|", np.abs(want).max())
    print(" got[:3,:3,0]", got[:3,:3,0])
    print(" want[:3,:3,0]", want[:3,:3,0])
    nz = np.nonzero(np.abs(got) > 0)
    print(" nonzero count", len(nz[0]), "of", got.size)
