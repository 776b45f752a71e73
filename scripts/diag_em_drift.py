"""Per-step parameter drift of the device EM step vs the fp64 oracle."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2004_06231_b200 as E
from paper_2004_06231_b200 import engine, trainer
from tests.test_gpu_tc import _pd_model
from oracle import einet_oracle as O


def rel(a, b, floor):
    return float(np.max(np.abs(a - b) / (np.abs(b) + floor)))


for tc in (True, False):
    circuit, fam, x, op = _pd_model(40, seed=3, both=False)
    engine.get_engine(circuit, fam, len(x)).set_tensor_cores(tc)
    model = E.EinetModel(circuit, engine.Parameters.from_numpy(circuit, fam, op.einsum,
                                                               op.mixing, op.phi), fam)
    for step in range(6):
        want_ll, op = O.em_step(circuit, op, fam.to_dict(), x, 0.5)
        ll = trainer.em_stochastic_step(model, x, 0.5)
        e2, m2, phi2 = model.params.to_numpy()
        werr = {i: rel(e2[i], op.einsum[i], 1e-9) for i in e2}
        print(f"tc={tc} step {step+1}: ll rel {abs(ll-want_ll)/abs(want_ll):.2e} "
              f"W {', '.join(f'{i}:{v:.1e}' for i, v in werr.items())} "
              f"mix {max([rel(m2[i], op.mixing[i], 1e-9) for i in m2] or [0]):.1e} "
              f"phi {rel(phi2, op.phi, 1e-9):.1e}", flush=True)
