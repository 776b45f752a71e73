"""C5 EinsumLayer sweep (BASELINE.json configs[4]): one
EinsumLayer of L = 64 rows with K_out = K, K in {10, 20, 40, 64, 128},
batch B in {64, ..., 4096}; forward and the two backward GEMMs (W statistics,
child responsibilities) timed separately, each against the tensor-core and the
HBM roofline.

    python scripts/sweep_c5.py [--out profiles/r02_c5_sweep.jsonl]

Graph: random_binary_tree(16 vars, depth 2, 32 replicas) -- the layer above
the leaves has exactly 2 x 32 = 64 product rows with K_out = K (the root layer,
32 rows with K_out = 1, and the mixing layer are not counted). Times are the
library's per-layer CUDA-event classes (EINET_PROFILE_LAYERS=1,
einet_profile_*), averaged over the repetitions of an uncaptured EM step:
`fwd` = the contraction (log-einsum-exp) launch(es) of the layer, `prep` = its
operand preparation (max-shift, exponentials, bf16 operand tiles), `wstats` and
`childrho` the two backward GEMMs (+ their fixed-order batch reductions).

Work per point: flops = 2 * B * L * K^3 per pass (forward,
W statistics; the child responsibilities are two such GEMMs, left and right);
bytes = 4 * (3 * B * L * K + L * K^3) per layer call (the two child
log-density vectors in, the output out, the weights). Peaks from
MEASURED_PEAKS.json (bf16 dense, HBM). K % 8 == 0 and K <= 64, K = 10, 20, 96, 128 run the
tcgen05 kernels (3xBF16: three MMAs per product, so `tc_frac_issued` = 3 x the
algorithmic fraction), the other K the CUDA-core kernels.
"""

import argparse
import json
import os
import sys

import numpy as np
import torch

os.environ["EINET_PROFILE_LAYERS"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2004_06231_b200 import _native, engine, trainer  # noqa: E402
from paper_2004_06231_b200.builders import make_family  # noqa: E402
from paper_2004_06231_b200.compiler import compile_graph  # noqa: E402
from paper_2004_06231_b200.model import EinetModel  # noqa: E402
from paper_2004_06231_b200.structures import StructureConfig, random_binary_tree  # noqa: E402

L_ROWS = 64


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
    except OSError:
        d = {}
    hbm = d.get("hbm_gbs") or d.get("hbm_copy_gbs") or 6543.7
    bf16 = d.get("bf16_tflops") or d.get("bf16_dense_tflops") or 1634.5
    return float(hbm), float(bf16)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ks", default="10,20,40,64,128")
    ap.add_argument("--batches", default="64,128,256,512,1024,2048,4096")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    hbm, bf16 = peaks()
    fam = make_family("gaussian", image_mode=False)
    rg = random_binary_tree(16, StructureConfig(depth=2, replicas=L_ROWS // 2, seed=0))
    rng = np.random.default_rng(0)
    lines = []
    for k in [int(v) for v in args.ks.split(",")]:
        circuit = compile_graph(rg, k)
        layer = [i for i, l in enumerate(circuit.layers)
                 if i > 0 and type(l).__name__ == "EinsumLayer" and len(l.left_src) == L_ROWS and l.k_out == k]
        assert layer, "no 64-row EinsumLayer with K_out = K"
        li = layer[0]
        x_all = rng.normal(0.0, 1.0, size=(max(int(b) for b in args.batches.split(",")), 16))
        ein, mix, phi = engine.init_parameters_host(circuit, fam, seed=0, data=x_all[:256])
        params = engine.Parameters.from_numpy(circuit, fam, ein, mix, phi)
        model = EinetModel(circuit, params, fam)
        tc = (k % 8 == 0 and 8 <= k <= 64) or k in (10, 20, 96, 128)
        for b in [int(v) for v in args.batches.split(",")]:
            xd = engine.as_device_batch(x_all[:b])
            for _ in range(3):
                trainer.em_stochastic_step(model, xd, 0.0)
            torch.cuda.synchronize()
            _native.profile_enable(True)
            for _ in range(args.reps):
                trainer.em_stochastic_step(model, xd, 0.0)
            torch.cuda.synchronize()
            prof = _native.profile_read()
            _native.profile_enable(False)
            us = {c: prof[f"{c}@{li}"][0] / args.reps * 1e3
                  for c in ("einsum_prep", "einsum_fwd", "einsum_wstats", "einsum_childrho")}
            flops = 2.0 * b * L_ROWS * k ** 3
            nbytes = 4.0 * (3 * b * L_ROWS * k + L_ROWS * k ** 3)
            line = {"k": k, "batch": b, "rows": L_ROWS, "k_out": k,
                    "path": "tcgen05 3xBF16" if tc else "CUDA cores fp32",
                    "ai_flop_per_byte": flops / nbytes}
            for name, c, mult in (("fwd", "einsum_fwd", 1), ("wstats", "einsum_wstats", 1),
                                  ("childrho", "einsum_childrho", 2)):
                t = us[c] * 1e-6
                tf = mult * flops / t / 1e12
                gbs = nbytes / t / 1e9
                line[f"{name}_us"] = us[c]
                line[f"{name}_tflops"] = tf
                line[f"{name}_tc_frac"] = tf / bf16
                line[f"{name}_tc_frac_issued"] = 3 * tf / bf16 if tc else None
                line[f"{name}_hbm_frac"] = gbs / hbm
            line["prep_us"] = us["einsum_prep"]
            line["fwd_with_prep_us"] = us["einsum_prep"] + us["einsum_fwd"]
            line["bound"] = "hbm" if flops / nbytes < bf16 * 1e3 / hbm else "tensor"
            print(json.dumps(line), flush=True)
            lines.append(line)
        del model, params
        torch.cuda.empty_cache()
    if args.out:
        with open(args.out, "w") as f:
            for line in lines:
                f.write(json.dumps(line) + "\n")


if __name__ == "__main__":
    main()
