"""C3 at B=64: device statistics and per-step parameters vs the fp64 oracle
(max relative error per block), tensor cores on/off. Diagnostics only."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2004_06231_b200 as E
from paper_2004_06231_b200 import engine, trainer
from paper_2004_06231_b200.data import config
from oracle import einet_oracle as O


def rel(a, b, atol):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b) / (atol + np.abs(b))))


rg, fam, k, gen = config("C3")
circuit = E.compile_graph(rg, k)
x = gen(64, seed=5).astype(np.float32).astype(np.float64)
ein, mix, phi = engine.init_parameters_host(circuit, fam, seed=0, data=x)
f32 = lambda a: np.asarray(a, np.float32).astype(np.float64)
op0 = O.OracleParams({i: f32(w) for i, w in ein.items()}, {i: f32(w) for i, w in mix.items()}, f32(phi))
for tc in (1, 0):
    op = op0
    p = engine.Parameters.from_numpy(circuit, fam, op.einsum, op.mixing, op.phi)
    eng = engine.get_engine(circuit, fam, len(x))
    eng.set_tensor_cores(tc)
    tr = engine.forward(circuit, p, fam, x)
    st = engine.backward(circuit, p, fam, tr)
    otr = O.forward(circuit, op, fam.to_dict(), x)
    ost = O.backward(circuit, op, fam.to_dict(), otr)
    print(f"tc={tc} stats: acc_pt {rel(st.acc_pt, ost.acc_pt, 1e-6 * 64):.2e} acc_p {rel(st.acc_p, ost.acc_p, 1e-6 * 64):.2e} "
          + " ".join(f"W{i} {rel(st.einsum[i], ost.einsum[i], 1e-6 * 64):.2e}" for i in st.einsum))
    model = E.EinetModel(circuit, p, fam)
    for step in range(3):
        want_ll, op = O.em_step(circuit, op, fam.to_dict(), x, 0.5)
        ll = trainer.em_stochastic_step(model, x, 0.5)
        e2, m2, phi2 = p.to_numpy()
        print(f"  step {step}: ll rel {abs(ll - want_ll) / abs(want_ll):.2e} phi {rel(phi2, op.phi, 1e-6):.2e} "
              + " ".join(f"W{i} {rel(e2[i], op.einsum[i], 1e-9):.2e}" for i in e2))
