"""Model and dataset files (reference ``modelio.py``), device-native.

EINM1 model files (``modelio.py:55-134``): magic ``EINM1``, u32 header
length, JSON header (region graph, k, k_root, family, replica assignment,
layer plan, provenance, tensor manifest), one blob per tensor (u32 ndim, u32
dims, little-endian f64 payload) in manifest order, closed by the zlib CRC32
of the blob section. The header is built and parsed on the host exactly like
the reference (same keys, same ``json.dumps``, so files are byte-identical);
the blob section moves between the file and the device parameters in one
copy, and the CRC32, the embedded-shape checks and the scatter/gather into
the flat fp64 parameter buffer run as CUDA kernels (csrc/io.cu:
``einet_crc32``, ``einet_params_from_blob``, ``einet_params_to_blob``).

EIND1 datasets (``modelio.py:137-187``): ``load_dataset`` / ``save_dataset``
with the reference's semantics; ``as_u8=True`` keeps a u8 payload as bytes
for the device decode path (``trainer.em_stochastic_steps``).
"""

from __future__ import annotations

import json
import struct

import numpy as np
import torch

from . import _native, engine
from .compiler import compile_graph
from .expfam import ExponentialFamily
from .model import EinetModel
from .structures import RegionGraph

MODEL_MAGIC = b"EINM1"
DATA_MAGIC = b"EIND1"
_INT32_MAX = 2 ** 31 - 1


class ModelFileError(ValueError):
    pass


class MagicError(ModelFileError):
    pass


class ChecksumError(ModelFileError):
    pass


class ShapeError(ModelFileError):
    pass


def _manifest(layout):
    """(name, parameter offset, shape) in the reference's tensor order
    (``modelio.py:42-47``: einsum layers, mixing layers, phi)."""
    out = [(f"einsum:{i}", off, tuple(shape)) for i, (off, shape) in sorted(layout.einsum.items())]
    out += [(f"mixing:{i}", off, tuple(shape))
            for i, (off, shape, _) in sorted(layout.mixing.items())]
    out.append(("phi", layout.phi_offset, tuple(layout.phi_shape)))
    return out


def _table(entries):
    """Device blob table rows {blob off, ndim, d0..d3, param off, count} and the
    blob length for (param offset or -1, shape) entries in blob order."""
    rows, off = [], 0
    for dst, shape in entries:
        if len(shape) > 4:
            raise ShapeError(f"tensor of rank {len(shape)} (at most 4 supported)")
        n = int(np.prod(shape)) if shape else 1
        dims = list(shape) + [0] * (4 - len(shape))
        rows.append([off, len(shape)] + dims + [dst, n])
        off += 4 + 4 * len(shape) + 8 * n
    return np.array(rows, dtype=np.int64).reshape(-1, 8), off


def _header(model):
    c = model.circuit
    return {
        "format": 1,
        "region_graph": json.loads(c.rg.to_json()),
        "k": c.k,
        "k_root": c.k_root,
        "family": model.family.to_dict(),
        "replica": {
            "count": c.replicas.count,
            "assignment": {str(k): v for k, v in sorted(c.replicas.replica_of.items())},
        },
        "layer_plan": json.loads(c.plan_json()),
        "provenance": model.provenance,
    }


def save_model(path, model: EinetModel):
    """Write an EINM1 file (reference ``modelio.py:50-79``): the parameters are
    gathered into the blob section and checksummed on the device, then copied
    to the host once."""
    lib = _native.lib()
    p = model.params
    man = _manifest(p._layout)
    header = _header(model)
    header["tensors"] = [{"name": n, "shape": list(s)} for n, _, s in man]
    hdr = json.dumps(header).encode("utf-8")
    table, blob_len = _table([(off, s) for _, off, s in man])
    dev = p.flat.device
    table_d = torch.from_numpy(table).to(dev)
    blob = torch.empty(blob_len + 4, dtype=torch.uint8, device=dev)
    crc = blob[blob_len:].view(torch.int32) if blob_len % 4 == 0 else \
        torch.empty(1, dtype=torch.int32, device=dev)
    st = engine._stream()
    _native.check(lib.einet_params_to_blob(engine._ptr(p.flat), engine._ptr(table_d),
                                           len(man), int(table[:, 7].max()),
                                           engine._ptr(blob), st), "einet_params_to_blob")
    _native.check(lib.einet_crc32(engine._ptr(blob), blob_len, engine._ptr(crc), st),
                  "einet_crc32")
    if crc.data_ptr() != blob.data_ptr() + blob_len:
        blob[blob_len:].copy_(crc.view(torch.uint8))
    host = blob.cpu().numpy()
    with open(path, "wb") as f:
        f.write(MODEL_MAGIC)
        f.write(struct.pack("<I", len(hdr)))
        f.write(hdr)
        f.write(host.tobytes())  # blob section + little-endian CRC32


def load_model(path, device=None) -> EinetModel:
    """Read an EINM1 file straight into device parameters (reference
    ``modelio.py:82-134``, same exceptions): one host->device copy of the blob
    section, CRC32 and per-tensor shape checks on the device."""
    raw = np.fromfile(path, dtype=np.uint8)
    if raw[:5].tobytes() != MODEL_MAGIC:
        raise MagicError(f"{path}: not a model file (bad magic)")
    if raw.size < 9:
        raise ChecksumError(f"{path}: truncated file")
    (hlen,) = struct.unpack_from("<I", raw, 5)
    header = json.loads(raw[9:9 + hlen].tobytes().decode("utf-8"))
    if raw.size < 9 + hlen + 4:
        raise ChecksumError(f"{path}: truncated file")
    blob_len = raw.size - 9 - hlen - 4
    (crc_want,) = struct.unpack_from("<I", raw, raw.size - 4)

    rg = RegionGraph.from_json(json.dumps(header["region_graph"]))
    circuit = compile_graph(rg, k=header["k"], k_root=header["k_root"])
    family = ExponentialFamily.from_dict(header["family"])
    layout = engine._Layout.of(circuit, family)
    dst = {n: (off, s) for n, off, s in _manifest(layout)}
    entries, names, seen = [], [], set()
    for spec in header["tensors"]:
        name, shape = spec["name"], tuple(int(v) for v in spec["shape"])
        off = -1
        if name in dst:
            off, want = dst[name]
            if shape != want:
                raise ShapeError(f"{path}: tensor {name}: header shape {list(shape)} "
                                 f"does not match the circuit {list(want)}")
            seen.add(name)
        entries.append((off, shape))
        names.append(name)
    for name in dst:
        if name not in seen:
            what = name.split(":")
            if len(what) == 2:
                raise ShapeError(f"{path}: missing weights for {what[0]} layer {what[1]}")
            raise ShapeError(f"{path}: missing tensor {name}")
    table, _ = _table(entries)

    _native.require_cuda()
    dev = device or torch.device("cuda", torch.cuda.current_device())
    lib = _native.lib()
    st = engine._stream()
    host = torch.from_numpy(raw[9 + hlen:9 + hlen + blob_len])
    if torch.cuda.is_available():
        host = host.pin_memory()
    blob = host.to(dev, non_blocking=True)
    table_d = torch.from_numpy(table).to(dev)
    flat = torch.zeros(layout.total, dtype=torch.float64, device=dev)
    words = torch.tensor([0, _INT32_MAX], dtype=torch.int32, device=dev)
    _native.check(lib.einet_crc32(engine._ptr(blob), blob_len, engine._ptr(words), st),
                  "einet_crc32")
    _native.check(lib.einet_params_from_blob(engine._ptr(blob), blob_len, engine._ptr(table_d),
                                             len(entries), int(table[:, 7].max(initial=0)),
                                             engine._ptr(flat), engine._ptr(words[1:]), st),
                  "einet_params_from_blob")
    crc_got, bad = [int(v) for v in words.cpu().tolist()]
    if (crc_got & 0xFFFFFFFF) != crc_want:
        raise ChecksumError(f"{path}: checksum mismatch (corrupt or truncated)")
    if bad != _INT32_MAX:
        e = table[bad]
        if e[0] + 4 + 4 * e[1] + 8 * e[7] > blob_len:
            raise ShapeError(f"{path}: blob section ends inside {names[bad]}")
        raise ShapeError(f"{path}: tensor {names[bad]}: header shape "
                         f"{list(entries[bad][1])} != blob shape")
    params = engine.Parameters(layout, flat)
    return EinetModel(circuit=circuit, params=params, family=family,
                      provenance=header.get("provenance", {}))


def load_dataset(path, normalize=None, as_u8=False) -> np.ndarray:
    """CSV or EIND1 binary (reference ``modelio.py:137-168``): float64 (n, d),
    u8 payloads divided by 255 by default. ``as_u8=True`` returns a u8
    payload as the raw (n, d) bytes instead, for the device decode path."""
    with open(path, "rb") as f:
        head = f.read(5)
    if head == DATA_MAGIC:
        raw = np.fromfile(path, dtype=np.uint8)
        n, d = struct.unpack_from("<II", raw, 5)
        tag = int(raw[13])
        payload = raw[14:]
        if tag == 0:
            arr = payload[:4 * n * d].view("<f4")
            if normalize is None:
                normalize = False
        elif tag == 1:
            arr = payload[:n * d]
            if as_u8:
                return arr.reshape(n, d).copy()
            if normalize is None:
                normalize = True
        else:
            raise ValueError(f"{path}: unknown dtype tag {tag}")
        data = arr.astype(np.float64).reshape(n, d)
    else:
        data = np.atleast_2d(np.loadtxt(path, delimiter=",", dtype=np.float64))
        if normalize is None:
            normalize = False
    if normalize:
        data = data / 255.0
    if data.size == 0:
        raise ValueError(f"{path}: empty dataset")
    return data


def save_dataset(path, data, dtype="f32"):
    """EIND1 writer (reference ``modelio.py:171-184``)."""
    data = np.atleast_2d(np.asarray(data))
    n, d = data.shape
    with open(path, "wb") as f:
        f.write(DATA_MAGIC)
        f.write(struct.pack("<II", n, d))
        if dtype == "f32":
            f.write(bytes([0]))
            f.write(np.ascontiguousarray(data, dtype="<f4").tobytes())
        elif dtype == "u8":
            f.write(bytes([1]))
            f.write(np.ascontiguousarray(data, dtype=np.uint8).tobytes())
        else:
            raise ValueError(f"unknown dtype {dtype!r}")
