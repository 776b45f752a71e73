"""Absolute error of device leaf rows / stats vs the fp64 oracle at init."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2004_06231_b200 import engine
from tests.test_gpu_tc import _pd_model
from oracle import einet_oracle as O

circuit, fam, x, op = _pd_model(40, seed=3, both=False)
p = engine.Parameters.from_numpy(circuit, fam, op.einsum, op.mixing, op.phi)
tr = engine.forward(circuit, p, fam, x)
rows = tr.leaf_rows
want = O.leaf_rows(circuit, fam.to_dict(), op.phi, x)
err = np.abs(rows - want)
print("leaf rows: |value| max %.3e  abs err max %.3e  mean %.3e" % (np.abs(want).max(), err.max(), err.mean()))
# error of the per-row differences to the row max (what the posterior sees)
d_got = rows - rows.max(axis=2, keepdims=True)
d_want = want - want.max(axis=2, keepdims=True)
near = d_want > -20
print("posterior-relevant offsets (> -20): abs err max %.3e" % np.abs(d_got - d_want)[near].max())
st = engine.backward(circuit, p, fam, tr)
otr = O.forward(circuit, op, fam.to_dict(), x)
ost = O.backward(circuit, op, fam.to_dict(), otr)
for i in ost.einsum:
    a, b = st.einsum[i], ost.einsum[i]
    print("W stats layer", i, "max rel (floor 1e-9) %.3e" % np.max(np.abs(a - b) / (np.abs(b) + 1e-9)))
a, b = st.acc_pt, ost.acc_pt
print("acc_pt max rel %.3e" % np.max(np.abs(a - b) / (np.abs(b) + 1e-9)))
a, b = st.acc_p, ost.acc_p
print("acc_p max rel %.3e" % np.max(np.abs(a - b) / (np.abs(b) + 1e-9)))
