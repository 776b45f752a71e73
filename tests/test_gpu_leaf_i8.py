"""The INT8 tensor-core leaf forward (csrc/leaf_i8.cu) at small sizes.

Batches below EINET_LEAF_I8_MIN_BATCH (default 1024) take the FP64 leaf path,
so the golden and randomised parity suites of test_gpu_parity.py would only
reach the INT8 kernel through the headline tests. Here the same suites run
with the INT8 path forced for every batch: image data on the 1/255 grid goes
through the integer tensor cores; off-grid data (the RAT Gaussian goldens,
NaN inputs) goes through the INT8 kernel, is flagged and falls back to the
FP64 path inside the same forward (conditional graph node / gated launches).
"""

import numpy as np
import pytest

from tests import test_gpu_parity as P
from tests.helpers import CASES

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def force_i8(monkeypatch):
    monkeypatch.setenv("EINET_LEAF_I8_MIN_BATCH", "0")


@pytest.mark.parametrize("name", CASES)
def test_forward_matches_reference_i8(name):
    P.test_forward_matches_reference(name)


@pytest.mark.parametrize("name", [c for c in CASES if c not in P.FULL_BATCH_SKIP])
def test_em_steps_match_reference_i8(name):
    P.test_em_steps_match_reference(name)


@pytest.mark.parametrize("seed", range(8))
def test_random_tensor_core_paths_vs_oracle_i8(seed):
    P.test_random_tensor_core_paths_vs_oracle(seed)


def test_c3_full_batch_vs_oracle_i8():
    P.test_c3_full_batch_vs_oracle()


def test_unsupported_values_raise_i8():
    P.test_unsupported_values_raise()
    P.test_unsupported_values_raise_dmma_path()


def test_training_is_deterministic_i8():
    P.test_training_is_deterministic()


@pytest.mark.parametrize("name,query,evidence", P.COND_CASES)
def test_conditional_log_density_matches_oracle_i8(name, query, evidence):
    P.test_conditional_log_density_matches_oracle(name, query, evidence)


def test_grid_values_evaluated_at_u_over_255():
    """A batch on the 1/255 grid and the same batch nudged one ulp off it:
    the first takes the INT8 path (values u / 255), the second the FP64
    fallback (fp32 values as given); both match the oracle fed the values
    each path evaluates."""
    import paper_2004_06231_b200 as E
    from paper_2004_06231_b200 import engine
    from paper_2004_06231_b200.data import config
    from oracle import einet_oracle as O
    from tests.helpers import device_values

    rg, fam, k, gen = config("C2")
    circuit = E.compile_graph(rg, k)
    x32 = gen(64, seed=5).astype(np.float32)
    ein, mix, phi = engine.init_parameters_host(circuit, fam, seed=0, data=x32.astype(np.float64))
    p = engine.Parameters.from_numpy(circuit, fam, ein, mix, phi)
    op = O.OracleParams(ein, mix, phi)
    off = x32.copy()
    off[3, 7] = np.nextafter(off[3, 7], np.float32(2))
    for xb in (x32, off):
        ll = E.forward(circuit, p, fam, xb).log_likelihood
        want = O.forward(circuit, op, fam.to_dict(), device_values(xb)).root[:, 0]
        assert np.all(np.abs(ll - want) <= 1e-4 * np.maximum(np.abs(want), 1.0))
