"""EINM1 model files and EIND1 datasets (reference modelio.py).

CPU: the header our writer builds is byte-identical to the files written by
the reference's own save_model (tests/golden/*.einm, gen_modelio.py), the
blob table reproduces the reference's blob layout, datasets round-trip.
GPU: files load straight into device parameters equal to the reference's,
saving reproduces the reference's file byte for byte, and corruption raises
the reference's exceptions.
"""

import ctypes
import json
import os
import struct
import types
import zlib

import numpy as np
import pytest

from paper_2004_06231_b200 import engine, modelio
from paper_2004_06231_b200.compiler import compile_graph
from paper_2004_06231_b200.expfam import ExponentialFamily
from paper_2004_06231_b200.structures import RegionGraph

from tests.helpers import GOLDEN, Case

FILES = ["rat_gaussian", "rat_categorical4", "pd_lift_gaussian_image", "rat_binomial"]


def read(name):
    with open(os.path.join(GOLDEN, name + ".einm"), "rb") as f:
        raw = f.read()
    (hlen,) = struct.unpack_from("<I", raw, 5)
    return raw, hlen, json.loads(raw[9:9 + hlen])


@pytest.mark.parametrize("name", FILES)
def test_header_is_byte_identical_to_reference(name):
    raw, hlen, header = read(name)
    rg = RegionGraph.from_json(json.dumps(header["region_graph"]))
    circuit = compile_graph(rg, header["k"], header["k_root"])
    family = ExponentialFamily.from_dict(header["family"])
    m = types.SimpleNamespace(circuit=circuit, family=family, provenance=header["provenance"])
    mine = modelio._header(m)
    layout = engine._Layout.of(circuit, family)
    man = modelio._manifest(layout)
    mine["tensors"] = [{"name": n, "shape": list(s)} for n, _, s in man]
    assert json.dumps(mine).encode("utf-8") == raw[9:9 + hlen]
    # the blob table reproduces the reference blob layout
    table, blob_len = modelio._table([(off, s) for _, off, s in man])
    assert blob_len == len(raw) - 9 - hlen - 4
    blob = raw[9 + hlen:-4]
    for row, (_, _, shape) in zip(table, man):
        off, ndim = int(row[0]), int(row[1])
        assert struct.unpack_from("<I", blob, off)[0] == ndim == len(shape)
        assert list(struct.unpack_from(f"<{ndim}I", blob, off + 4)) == list(shape)
    assert zlib.crc32(blob) == struct.unpack_from("<I", raw, len(raw) - 4)[0]


def test_dataset_round_trip(tmp_path):
    rng = np.random.default_rng(0)
    x = rng.random((7, 5))
    p = str(tmp_path / "a.eind")
    modelio.save_dataset(p, x)
    assert np.array_equal(modelio.load_dataset(p), x.astype(np.float32).astype(np.float64))
    u = rng.integers(0, 256, (6, 4)).astype(np.uint8)
    modelio.save_dataset(p, u, dtype="u8")
    assert np.array_equal(modelio.load_dataset(p), u / 255.0)
    assert np.array_equal(modelio.load_dataset(p, normalize=False), u.astype(np.float64))
    raw = modelio.load_dataset(p, as_u8=True)
    assert raw.dtype == np.uint8 and np.array_equal(raw, u)
    c = str(tmp_path / "b.csv")
    np.savetxt(c, x, delimiter=",")
    assert np.allclose(modelio.load_dataset(c), x)
    with pytest.raises(ValueError):
        modelio.save_dataset(p, x, dtype="f16")


# ---------------------------------------------------------------------------
# device paths
# ---------------------------------------------------------------------------

@pytest.mark.gpu
@pytest.mark.parametrize("name", FILES)
def test_load_matches_reference_and_save_is_byte_identical(name, tmp_path):
    case = Case(name)
    m = modelio.load_model(os.path.join(GOLDEN, name + ".einm"))
    ein, mix, phi = m.params.to_numpy()
    want = case.params("init")
    for i in want.einsum:
        assert np.array_equal(ein[i], want.einsum[i])
    for i in want.mixing:
        assert np.array_equal(mix[i], want.mixing[i])
    assert np.array_equal(phi, want.phi)
    out = str(tmp_path / "m.einm")
    modelio.save_model(out, m)
    with open(out, "rb") as f, open(os.path.join(GOLDEN, name + ".einm"), "rb") as g:
        assert f.read() == g.read()
    # the loaded model runs: LL equals a model built from the same arrays
    p = engine.Parameters.from_numpy(case.circuit, case.family, want.einsum, want.mixing,
                                     want.phi)
    a = engine.forward(m.circuit, m.params, m.family, case.x).log_likelihood
    b = engine.forward(case.circuit, p, case.family, case.x).log_likelihood
    assert np.array_equal(a, b)


@pytest.mark.gpu
def test_corrupt_files_raise_reference_errors(tmp_path):
    raw, hlen, header = read("rat_gaussian")
    p = str(tmp_path / "x.einm")

    def write(b):
        with open(p, "wb") as f:
            f.write(b)

    write(b"EINM2" + raw[5:])
    with pytest.raises(modelio.MagicError):
        modelio.load_model(p)
    bad = bytearray(raw)
    bad[9 + hlen + 100] ^= 0x10
    write(bytes(bad))
    with pytest.raises(modelio.ChecksumError):
        modelio.load_model(p)
    write(raw[:-40])
    with pytest.raises(modelio.ChecksumError):
        modelio.load_model(p)
    # an embedded dim that disagrees with the manifest, checksum recomputed
    blob = bytearray(raw[9 + hlen:-4])
    struct.pack_into("<I", blob, 4, 999)
    write(raw[:9 + hlen] + bytes(blob) + struct.pack("<I", zlib.crc32(bytes(blob))))
    with pytest.raises(modelio.ShapeError):
        modelio.load_model(p)
    # a manifest without the leaf tensor
    h = dict(header)
    h["tensors"] = [t for t in header["tensors"] if t["name"] != "phi"]
    hb = json.dumps(h).encode()
    write(raw[:5] + struct.pack("<I", len(hb)) + hb + raw[9 + hlen:])
    with pytest.raises(modelio.ShapeError):
        modelio.load_model(p)


@pytest.mark.gpu
def test_device_crc32_matches_zlib():
    import torch
    from paper_2004_06231_b200 import _native
    rng = np.random.default_rng(1)
    lib = _native.lib()
    for n in (0, 1, 3, 1023, 1024, 1025, 262143, 262144 + 17, 9_000_001):
        a = rng.integers(0, 256, n + 3).astype(np.uint8)
        d = torch.from_numpy(a).cuda()
        crc = torch.zeros(1, dtype=torch.int32, device="cuda")
        for lo in (0, 3):  # aligned and unaligned starts
            _native.check(lib.einet_crc32(ctypes.c_void_p(d.data_ptr() + lo), n, engine._ptr(crc),
                                          engine._stream()), "crc")
            assert (int(crc.item()) & 0xFFFFFFFF) == zlib.crc32(a[lo:lo + n].tobytes()), (n, lo)


@pytest.mark.gpu
def test_save_load_round_trip_c3(tmp_path):
    from paper_2004_06231_b200 import trainer
    from paper_2004_06231_b200.data import config
    from paper_2004_06231_b200.model import build_model
    rg, fam, k, gen = config("C3")
    x = gen(256, seed=2)
    m = build_model(rg, fam, k=k, seed=0, data=x, provenance={"epochs": 1})
    trainer.em_stochastic_step(m, x, 0.5)
    p = str(tmp_path / "c3.einm")
    modelio.save_model(p, m)
    back = modelio.load_model(p)
    import torch
    assert torch.equal(back.params.flat, m.params.flat)
    assert back.provenance == {"epochs": 1}
    assert np.array_equal(back.log_likelihood(x), m.log_likelihood(x))
