"""C3 at B=64: tensor-core leaf statistics vs the oracle, error pattern. Diagnostics only."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2004_06231_b200 as E
from paper_2004_06231_b200 import engine
from paper_2004_06231_b200.data import config
from oracle import einet_oracle as O

rg, fam, k, gen = config("C3")
circuit = E.compile_graph(rg, k)
x = gen(64, seed=5).astype(np.float32).astype(np.float64)
ein, mix, phi = engine.init_parameters_host(circuit, fam, seed=0, data=x)
f32 = lambda a: np.asarray(a, np.float32).astype(np.float64)
op = O.OracleParams({i: f32(w) for i, w in ein.items()}, {i: f32(w) for i, w in mix.items()}, f32(phi))
otr = O.forward(circuit, op, fam.to_dict(), x)
ost = O.backward(circuit, op, fam.to_dict(), otr)
want = ost.acc_pt  # (D, K, R, 2)
for tc in (1, 0):
    p = engine.Parameters.from_numpy(circuit, fam, op.einsum, op.mixing, op.phi)
    eng = engine.get_engine(circuit, fam, len(x))
    eng.set_tensor_cores(tc)
    tr = engine.forward(circuit, p, fam, x)
    st = engine.backward(circuit, p, fam, tr)
    got = st.acc_pt
    err = np.abs(got - want)
    scale = np.abs(want).max(axis=(0, 1, 2), keepdims=True)
    print(f"tc={tc}: max abs err t0 {err[..., 0].max():.3e} t1 {err[..., 1].max():.3e}; "
          f"max |want| t0 {np.abs(want[..., 0]).max():.3e} t1 {np.abs(want[..., 1]).max():.3e}")
    e = err[..., 1] / (1e-9 + np.abs(want[..., 1]))
    idx = np.unravel_index(np.argsort(e.ravel())[-5:], e.shape)
    for d, kk, r in zip(*idx):
        print(f"   d={d} k={kk} r={r}: got {got[d, kk, r]} want {want[d, kk, r]}")
    bad = (err[..., 1] > 1e-4 * np.abs(want[..., 1]) + 1e-7)
    ds = np.nonzero(bad.any(axis=(1, 2)))[0]
    print("   bad d count", len(ds), "first", ds[:20], "mod 4", np.bincount(ds % 4, minlength=4))

wp = ost.acc_p
for tc in (1, 0):
    p = engine.Parameters.from_numpy(circuit, fam, op.einsum, op.mixing, op.phi)
    eng = engine.get_engine(circuit, fam, len(x))
    eng.set_tensor_cores(tc)
    tr = engine.forward(circuit, p, fam, x)
    st = engine.backward(circuit, p, fam, tr)
    gp = st.acc_p
    e = np.abs(gp - wp)
    i = np.unravel_index(np.argmax(e), e.shape)
    print(f"tc={tc}: acc_p max abs err {e.max():.3e} at {i}: got {gp[i]} want {wp[i]}")
    # implied S error for the worst acc_pt entry
    ga = st.acc_pt
    d, kk, r = 258, 5, 0
    print(f"   d=258 k=5: P got {gp[d, kk, r]:.3e} want {wp[d, kk, r]:.3e}; acc_pt got {ga[d, kk, r]} want {want[d, kk, r]}")
