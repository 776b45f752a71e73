"""Speed of the oracle port (the reference arm of bench.py) against the
reference's own EM step on the same host, same C3 sample, same core count.

Run in the build container only (the reference exists only here):
    python scripts/port_vs_reference.py [N] [REPS]
It times one `trainer.em_stochastic_step` (/root/reference/pkg/src/einet/
trainer.py:99-117) of the reference on N C3 samples, single-threaded BLAS, and
the same update through `oracle.einet_oracle.em_step` (bench.py's CPU legs),
then checks the two updates agree (mean LL, parameters). Output: one JSON
line (profiles/r02_port_vs_reference.json).
"""
import json
import os
import sys
import time

for v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ[v] = "1"

import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))

from gen_golden import _ref, lift3  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 96
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    builders, compiler, engine, expfam, model, structures, trainer = _ref()
    from paper_2004_06231_b200 import engine as E
    from paper_2004_06231_b200.compiler import compile_graph
    from paper_2004_06231_b200.data import config
    from oracle import einet_oracle as O

    S = structures
    rg_ref = lift3(S, S.poon_domingos(32, 32, S.StructureConfig(deltas=(8,), axes="vertical")))
    rg, fam, k, gen = config("C3")
    x = gen(n, seed=0).astype(np.float32).astype(np.float64)
    m = model.build_model(rg_ref, builders.make_family("gaussian", image_mode=True), k=k,
                          seed=0, data=x)
    circuit = compile_graph(rg, k)
    ein, mix, phi = E.init_parameters_host(circuit, fam, seed=0, data=x)
    assert np.array_equal(phi, m.params.phi), "init differs from the reference"

    def t_ref():
        t0 = time.perf_counter()
        ll = trainer.em_stochastic_step(m, x, 0.5)
        return time.perf_counter() - t0, ll

    p = O.OracleParams(ein, mix, phi)
    fd = fam.to_dict()
    state = {"p": p}

    def t_port():
        t0 = time.perf_counter()
        ll, p_new = O.em_step(circuit, state["p"], fd, x, 0.5)
        return time.perf_counter() - t0, (p_new, ll)

    r0, ll_ref0 = t_ref()
    q0, (p1, ll_port0) = t_port()
    phi_ref = m.params.phi.copy()
    rel = float(np.max(np.abs(p1.phi - phi_ref) / np.maximum(np.abs(phi_ref), 1e-12)))
    tr, tp = [], []
    for _ in range(reps):
        tr.append(t_ref()[0])
        tp.append(t_port()[0])
    ref_s, port_s = float(np.median(tr)), float(np.median(tp))
    print(json.dumps({
        "config": "C3 SVHN-shape PD K=40, EM lambda 0.5", "samples_per_step": n, "reps": reps,
        "cores": 1, "reference_s_per_step": ref_s, "port_s_per_step": port_s,
        "reference_samples_per_s": n / ref_s, "port_samples_per_s": n / port_s,
        "port_over_reference": ref_s / port_s,
        "first_step_mean_ll": {"reference": float(ll_ref0), "port": float(ll_port0)},
        "first_step_phi_max_rel_diff": rel}))


if __name__ == "__main__":
    main()
