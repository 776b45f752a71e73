"""einet_pack_f64 (host-only C-ABI entry, no device call): the float64 batch a
reference caller passes (trainer.py:104; image datasets are v / 255 in
float64, modelio.py:145-166) is packed to one byte per value when it lies on
the u8 grid, else to fp32 -- and the fp32 values the engine then sees equal
the host cast of the batch either way."""

import ctypes

import numpy as np
import pytest


def pack(lib, x, with_f32=True, threads=0):
    x = np.ascontiguousarray(x, dtype=np.float64)
    u8 = np.zeros(x.size, np.uint8)
    f32 = np.zeros(x.size, np.float32)
    kind = ctypes.c_int32(-7)
    rc = lib.einet_pack_f64(x.ctypes.data, x.size, u8.ctypes.data,
                            f32.ctypes.data if with_f32 else None, threads, ctypes.byref(kind))
    assert rc == 0
    return kind.value, u8, f32


def decoded(kind, u8, f32):
    """fp32 values the device sees (k_decode_u8: (float)((double)v / divisor))."""
    if kind == 0:
        return f32
    return (u8.astype(np.float64) / float(kind)).astype(np.float32)


@pytest.mark.parametrize("n", [0, 1, 4095, 4097, 3 * (1 << 18) + 5])
def test_image_grid_packs_to_bytes(native_lib, n):
    rng = np.random.default_rng(n)
    v = rng.integers(0, 256, n)
    x = v / 255.0
    kind, u8, f32 = pack(native_lib, x)
    assert kind == 255
    assert np.array_equal(u8, v.astype(np.uint8))
    assert np.array_equal(decoded(kind, u8, f32).view(np.uint32),
                          x.astype(np.float32).view(np.uint32))


def test_raw_counts_pack_to_bytes(native_lib):
    v = np.random.default_rng(1).integers(0, 4, 10000)
    kind, u8, f32 = pack(native_lib, v.astype(np.float64))
    assert kind == 1 and np.array_equal(u8, v.astype(np.uint8))


def test_binary_data_is_on_the_image_grid(native_lib):
    v = np.random.default_rng(2).integers(0, 2, 1000).astype(np.float64)
    kind, u8, f32 = pack(native_lib, v)
    assert kind == 255
    assert np.array_equal(decoded(kind, u8, f32), v.astype(np.float32))


@pytest.mark.parametrize("bad", [np.nan, np.inf, -np.inf, -0.0, -1 / 255, 256 / 255, 0.5,
                                 1.0 / 255 + 1e-17 * 0 + np.spacing(1.0 / 255)])
@pytest.mark.parametrize("pos", [0, 777, 2_000_000 - 1])
def test_off_grid_values_give_fp32(native_lib, bad, pos):
    x = np.random.default_rng(3).integers(0, 256, 2_000_000) / 255.0
    x[pos] = bad
    kind, u8, f32 = pack(native_lib, x)
    assert kind == 0
    assert np.array_equal(f32.view(np.uint32), x.astype(np.float32).view(np.uint32))
    kind, _, _ = pack(native_lib, x, with_f32=False)
    assert kind == -1


def test_gaussian_data_gives_fp32_on_any_thread_count(native_lib):
    x = np.random.default_rng(4).normal(size=1_500_000)
    for t in (1, 3, 0):
        kind, u8, f32 = pack(native_lib, x, threads=t)
        assert kind == 0
        assert np.array_equal(f32, x.astype(np.float32))


def test_bad_arguments(native_lib):
    kind = ctypes.c_int32()
    assert native_lib.einet_pack_f64(None, -1, None, None, 0, ctypes.byref(kind)) != 0
    assert native_lib.einet_pack_f64(None, 5, None, None, 0, ctypes.byref(kind)) != 0
    assert native_lib.einet_pack_f64(None, 0, None, None, 0, None) != 0
