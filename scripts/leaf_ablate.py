"""Leaf-forward timing on C3 at B=16384 (diagnostic): per-class device time
of `forward` for the INT8 path under EINET_I8_DEBUG ablations and for the
FP64 path (EINET_LEAF_I8=0). Each setting runs in its own process."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def one():
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch
    import paper_2004_06231_b200 as E
    from paper_2004_06231_b200 import _native, engine
    from paper_2004_06231_b200.data import config
    B = int(os.environ.get("ABL_B", "16384"))
    rg, fam, k, gen = config(os.environ.get("ABL_CFG", "C3"))
    circuit = E.compile_graph(rg, k)
    x = torch.from_numpy(gen(B, seed=3).astype(np.float32)).cuda()
    ein, mix, phi = engine.init_parameters_host(circuit, fam, seed=0, data=gen(512, seed=1))
    p = engine.Parameters.from_numpy(circuit, fam, ein, mix, phi)
    for _ in range(3):
        E.forward(circuit, p, fam, x)
    torch.cuda.synchronize()
    _native.profile_enable(True)
    n = 10
    for _ in range(n):
        E.forward(circuit, p, fam, x)
    torch.cuda.synchronize()
    prof = _native.profile_read()
    _native.profile_enable(False)
    print(json.dumps({k: v[0] / n * 1e3 for k, v in prof.items()}))


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "one":
        one()
        sys.exit(0)
    settings = [("i8", {}), ("i8 nofb", {"EINET_I8_DEBUG": "32"}),
                ("nofb noepi", {"EINET_I8_DEBUG": "34"}), ("nofb nomma", {"EINET_I8_DEBUG": "36"}),
                ("i8 B=500", {"ABL_B": "500"}), ("fp64 B=500", {"ABL_B": "500", "EINET_LEAF_I8": "0"}),
                ("fp64 dmma", {"EINET_LEAF_I8": "0"})]
    for name, env in settings:
        e = dict(os.environ, **env)
        out = subprocess.run([sys.executable, __file__, "one"], env=e, capture_output=True,
                             text=True, timeout=300)
        line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-400:]
        print(f"{name:16s} {line}", flush=True)
