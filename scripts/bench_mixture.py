"""Mixture-of-EiNets training throughput (paper section 4.2 pipeline, the
BASELINE.md SVHN row: 100-component PD EiNet mixture, K=40, delta 8 vertical,
batch 500, lambda 0.5; 5 h for 25 epochs of 581k images on a P100, ~810
samples/s derived).

    python scripts/bench_mixture.py [--components 100] [--per 5810] [--epochs 2]

Synthetic SVHN-shaped data, one cluster per component (k-means is host
preprocessing and is not timed). Epoch 0 captures the CUDA graphs and is not
timed; the timed epochs include every EM step and the per-epoch training-LL
pass of every component, like ``train_mixture``; the one-time upload of the
datasets to the device is reported separately. Prints one JSON line.
"""

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2004_06231_b200 import engine, trainer  # noqa: E402
from paper_2004_06231_b200.compiler import compile_graph  # noqa: E402
from paper_2004_06231_b200.data import config  # noqa: E402
from paper_2004_06231_b200.model import EinetModel  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--components", type=int, default=100)
    ap.add_argument("--per", type=int, default=5810)
    ap.add_argument("--epochs", type=int, default=2)
    ap.add_argument("--batch", type=int, default=500)
    ap.add_argument("--streams", type=int, default=16)
    args = ap.parse_args()
    rg, fam, k, gen = config("C3")
    circuit = compile_graph(rg, k)  # one compiled structure shared by all components
    datas = [gen(args.per, seed=100 + c) for c in range(args.components)]
    models = []
    for c, d in enumerate(datas):
        ein, mix, phi = engine.init_parameters_host(circuit, fam, seed=c, data=d[:512])
        models.append(EinetModel(circuit, engine.Parameters.from_numpy(circuit, fam, ein, mix,
                                                                       phi), fam))
    torch.cuda.synchronize()
    t = time.perf_counter()
    datas = [engine.as_device_batch(d) for d in datas]  # resident for all epochs
    torch.cuda.synchronize()
    upload = time.perf_counter() - t
    cfg = trainer.TrainerConfig(epochs=1, batch_size=args.batch, step_size=0.5, seed=0)
    t = time.perf_counter()
    trainer.train_many(models, datas, cfg, streams=args.streams)  # captures the graphs
    warm = time.perf_counter() - t
    cfg.epochs = args.epochs
    torch.cuda.synchronize()
    t = time.perf_counter()
    met = trainer.train_many(models, datas, cfg, streams=args.streams)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    n = args.components * args.per
    steps = args.components * -(-args.per // args.batch)
    print(json.dumps({
        "metric": "mixture EM training samples/s (SVHN-shape PD EiNet K=40 components)",
        "value": n * args.epochs / dt, "unit": "samples/s", "components": args.components,
        "samples_per_component": args.per, "batch": args.batch, "epochs_timed": args.epochs,
        "ms_per_epoch": dt / args.epochs * 1e3, "em_steps_per_epoch": steps,
        "us_per_em_step": dt / args.epochs / steps * 1e6, "streams": args.streams,
        "warmup_epoch_s": warm, "dataset_upload_s": upload, "mean_train_ll_last_epoch": float(np.mean(
            [m[-1].train_ll for m in met])),
        "paper_p100_derived": 810.0, "data": "synthetic",
    }))


if __name__ == "__main__":
    main()
