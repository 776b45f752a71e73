"""Generate EINM1 model files with the reference's own ``save_model``.

Run in the build container (the reference exists only here):
    python tests/golden/gen_modelio.py
For a few golden circuits (the fp32 ``init`` parameters of the .npz fixtures
made by gen_golden.py) it builds the reference model, sets a provenance
document and writes ``<case>.einm`` with ``modelio.save_model``
(modelio.py:50-79). tests/ check that paper_2004_06231_b200.modelio reads
these files into identical device parameters and writes byte-identical
files.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
CASES = ["rat_gaussian", "rat_categorical4", "pd_lift_gaussian_image", "rat_binomial"]


def provenance(name):
    return {"case": name, "source": "tests/golden/gen_modelio.py", "steps": 0}


def main():
    sys.path.insert(0, REF)
    from einet import compiler, engine, expfam, model, modelio, structures

    for name in CASES:
        z = dict(np.load(os.path.join(HERE, name + ".npz")))
        rg = structures.RegionGraph.from_json(str(z["rg_json"]))
        circuit = compiler.compile_graph(rg, int(z["k"]), int(z["k_root"]))
        family = expfam.ExponentialFamily.from_dict(json.loads(str(z["family_json"])))
        ein = {i: z[f"init_einsum_{i}"] for i, l in enumerate(circuit.layers)
               if type(l).__name__ == "EinsumLayer"}
        mix = {i: z[f"init_mixing_{i}"] for i, l in enumerate(circuit.layers)
               if type(l).__name__ == "MixingLayer"}
        params = engine.Parameters(einsum=ein, mixing=mix, phi=z["init_phi"])
        m = model.EinetModel(circuit=circuit, params=params, family=family,
                             provenance=provenance(name))
        path = os.path.join(HERE, name + ".einm")
        modelio.save_model(path, m)
        back = modelio.load_model(path)
        assert np.array_equal(back.params.phi, params.phi)
        print(name, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
