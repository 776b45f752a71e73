"""Measurements for the SURVEY.md 8f rows on the C3 model (SVHN-shaped PD,
K=40, 3072 variables): batched ancestral sampling, image-completion
conditional sampling (left half observed), conditional log-density of the
right half given the left half over a batch, and EINM1 save / load through
the device paths. Each GPU leg is timed end to end through the public API
(numpy results on the host), best of 3 after a warm-up; the sampling legs
also time the oracle's restatement of the reference's per-sample descent
(oracle.sample_philox, one host core) on a bounded sample. Also the plain
log-likelihood (forward) throughput from a device-resident and a numpy batch.

    python scripts/bench_widen.py [--out profiles/r01_widen_bench.json]
"""

import argparse
import json
import os
import sys
import tempfile
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2004_06231_b200 as E  # noqa: E402
from paper_2004_06231_b200 import engine, modelio  # noqa: E402
from paper_2004_06231_b200.data import config  # noqa: E402


def best_of(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(reps):
        t = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    from oracle import einet_oracle as O
    rg, fam, k, gen = config("C3")
    x = gen(16384, seed=3)
    m = E.build_model(rg, fam, k=k, seed=0, data=x[:4096])
    E.trainer.em_stochastic_steps(m, [x] * 3, 0.5)
    d = m.circuit.d_vars
    left = [v for v in range(d) if (v // 3) % 32 < 16]
    right = [v for v in range(d) if (v // 3) % 32 >= 16]
    out = {"model": "C3 SVHN-shape 32x32x3 PD EiNet K=40", "data": "synthetic"}

    n = 16384
    xd = engine.as_device_batch(x[:n])
    t = best_of(lambda: m.log_likelihood(xd, chunk=n))
    out["log_likelihood"] = {"batch": n, "input": "device-resident fp32", "s": t,
                             "samples_per_s": n / t}
    t = best_of(lambda: m.log_likelihood(x[:n], chunk=n))
    out["log_likelihood_numpy"] = {"batch": n, "input": "numpy float64", "s": t,
                                   "samples_per_s": n / t}
    t = best_of(lambda: m.sample(n, seed=1))
    out["sample"] = {"n": n, "s": t, "samples_per_s": n / t}
    n = 4096
    t = best_of(lambda: m.conditional_sample(x[0], left, n, seed=2))
    out["conditional_sample"] = {"n": n, "evidence": "left half (1536 variables)", "s": t,
                                 "samples_per_s": n / t}
    n = 16384
    t = best_of(lambda: m.conditional_log_density(x[:n], right, left))
    out["conditional_log_density"] = {"batch": n, "query": "right half", "evidence": "left half",
                                      "s": t, "samples_per_s": n / t}
    with tempfile.TemporaryDirectory() as tmp:
        path = os.path.join(tmp, "c3.einm")
        t_save = best_of(lambda: modelio.save_model(path, m))
        t_load = best_of(lambda: modelio.load_model(path))
        out["einm1"] = {"bytes": os.path.getsize(path), "save_s": t_save, "load_s": t_load}

    # oracle restatement of the reference descent, bounded sample, one core
    ein, mix, phi = m.params.to_numpy()
    op = O.OracleParams(ein, mix, phi)
    n_cpu = 64
    t = time.perf_counter()
    O.sample_philox(m.circuit, op, fam.to_dict(), n_cpu, seed=1)
    t = time.perf_counter() - t
    out["sample"]["cpu_oracle"] = {"n": n_cpu, "s": t, "samples_per_s": n_cpu / t, "cores": 1,
                                   "kind": "port (oracle.sample_philox)"}
    out["sample"]["speedup_vs_cpu_oracle"] = out["sample"]["samples_per_s"] / (n_cpu / t)
    line = json.dumps(out)
    print(line)
    if args.out:
        with open(args.out, "w") as f:
            f.write(line + "\n")


if __name__ == "__main__":
    main()
