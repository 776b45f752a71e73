"""EinsumLayer contraction sweep (BASELINE.json configs[4]): K in
{10, 20, 40, 64, 128} x batch in {64, 256, 1024, 4096} on the SVHN-shaped PD
graph (lifted 32x32x3, delta 8 vertical): the forward contraction and the two
back-pass GEMMs (W statistics, child responsibilities) of an EM step.

    python scripts/sweep_einsum.py [--out profiles/r01_einsum_sweep.json]

The EinsumLayer forward time per pass is the ``einsum_fwd`` class of the
library's CUDA-event profiler (einet_profile_*: the A-operand preparation,
the contraction and its epilogue, every einsum layer); work = 2 * sum_rows
K_out * K^2 flops per sample (the 'bip,bjp,ijop->bop' contraction), bytes =
the fp32 child offsets read and the output offsets written, (2K + K_out) * 4
per row and sample. K % 8 == 0 and K <= 64 run the tcgen05 kernels (3xBF16,
three MMAs per product), the others the CUDA-core kernels. One JSON object
per line.
"""

import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2004_06231_b200 import _native, engine, trainer  # noqa: E402
from paper_2004_06231_b200.model import EinetModel  # noqa: E402
from paper_2004_06231_b200.compiler import compile_graph  # noqa: E402
from paper_2004_06231_b200.data import config  # noqa: E402


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return d.get("hbm_gbs", 6650.0), d.get("bf16_tflops", 1590.0)
    except OSError:
        return 6650.0, 1590.0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ks", default="10,20,40,64,128")
    ap.add_argument("--batches", default="64,256,1024,4096")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    hbm, bf16 = peaks()
    rg, fam, _, gen = config("C3")
    lines = []
    for k in [int(v) for v in args.ks.split(",")]:
        circuit = compile_graph(rg, k)
        rows = [(len(l.left_src), l.k_out) for l in circuit.layers[1:]
                if type(l).__name__ == "EinsumLayer"]
        flops = sum(2 * r * ko * k * k for r, ko in rows)
        nbytes = sum(r * (2 * k + ko) * 4 for r, ko in rows)
        x_all = gen(max(int(b) for b in args.batches.split(",")), seed=1)
        ein, mix, phi = engine.init_parameters_host(circuit, fam, seed=0, data=x_all[:512])
        params = engine.Parameters.from_numpy(circuit, fam, ein, mix, phi)
        tc = k % 8 == 0 and 8 <= k <= 64
        for b in [int(v) for v in args.batches.split(",")]:
            xd = engine.as_device_batch(x_all[:b])
            for _ in range(3):
                engine.forward(circuit, params, fam, xd, check=False)
            torch.cuda.synchronize()
            _native.profile_enable(True)
            for _ in range(args.reps):
                engine.forward(circuit, params, fam, xd, check=False)
            torch.cuda.synchronize()
            prof = _native.profile_read()
            _native.profile_enable(False)
            ms = prof["einsum_fwd"][0] / args.reps
            tfs = flops * b / (ms / 1e3) / 1e12
            gbs = nbytes * b / (ms / 1e3) / 1e9
            # the back-pass GEMMs of one uncaptured EM step (W statistics: the
            # forward's flops; child responsibilities: twice them)
            model = EinetModel(circuit, params, fam)
            trainer.em_stochastic_step(model, xd, 0.0)
            torch.cuda.synchronize()
            _native.profile_enable(True)
            for _ in range(max(1, args.reps // 4)):
                trainer.em_stochastic_step(model, xd, 0.0)
            torch.cuda.synchronize()
            bprof = _native.profile_read()
            _native.profile_enable(False)
            nb = max(1, args.reps // 4)
            ws_ms = bprof["einsum_wstats"][0] / nb
            cr_ms = bprof["einsum_childrho"][0] / nb
            line = {"k": k, "batch": b, "path": "tcgen05 3xBF16" if tc else "CUDA cores fp32",
                    "einsum_fwd_us": ms * 1e3, "tflops": tfs, "gbs": gbs,
                    "frac_bf16_peak": tfs / bf16,
                    "frac_bf16_peak_3x": 3 * tfs / bf16 if tc else None,
                    "frac_hbm": gbs / hbm, "flops_per_sample": flops,
                    "bytes_per_sample": nbytes, "rows": rows,
                    "wstats_us": ws_ms * 1e3,
                    "wstats_tflops": flops * b / (ws_ms / 1e3) / 1e12,
                    "childrho_us": cr_ms * 1e3,
                    "childrho_tflops": 2 * flops * b / (cr_ms / 1e3) / 1e12}
            print(json.dumps(line), flush=True)
            lines.append(line)
        del params
        torch.cuda.empty_cache()
    if args.out:
        with open(args.out, "w") as f:
            for line in lines:
                f.write(json.dumps(line) + "\n")


if __name__ == "__main__":
    main()
