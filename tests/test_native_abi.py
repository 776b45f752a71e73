"""The C-ABI library: loads without a GPU, exports every entry point declared
in include/einet_b200.h, matches the ctypes struct layouts, and rejects bad
plans on the host before touching the device."""

import ctypes
import os
import re
import subprocess

import pytest

from paper_2004_06231_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "einet_b200.h")


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^[\w ]+?\*?\s*\b(einet_\w+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol(native_lib):
    names = declared_functions()
    assert len(names) >= 15
    for name in names:
        assert hasattr(native_lib, name), name
        assert name in _native.EXPORTS, f"{name} missing from the ctypes binding"


def test_struct_layouts_match_c(tmp_path, native_lib):
    src = tmp_path / "layout.c"
    src.write_text(r'''
#include <stddef.h>
#include <stdio.h>
#include "einet_b200.h"
#define F(T, m) printf(#T "." #m " %zu\n", offsetof(T, m));
int main(void) {
  printf("einet_layer_desc %zu\n", sizeof(einet_layer_desc));
  printf("einet_plan_desc %zu\n", sizeof(einet_plan_desc));
  printf("einet_sizes %zu\n", sizeof(einet_sizes));
  F(einet_layer_desc, left) F(einet_layer_desc, mask)
  F(einet_plan_desc, var_min) F(einet_plan_desc, n_leaf) F(einet_plan_desc, leaf_scope_offsets)
  F(einet_plan_desc, layers) F(einet_plan_desc, root_mix_row)
  F(einet_sizes, compute_bytes) F(einet_sizes, suff_dim)
  return 0;
}''')
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)],
                   check=True)
    got = dict(line.split() for line in subprocess.run([str(exe)], capture_output=True,
                                                        text=True, check=True).stdout.split("\n")
               if line)
    assert int(got["einet_layer_desc"]) == ctypes.sizeof(_native.LayerDesc)
    assert int(got["einet_plan_desc"]) == ctypes.sizeof(_native.PlanDesc)
    assert int(got["einet_sizes"]) == ctypes.sizeof(_native.Sizes)
    for key, value in got.items():
        if "." not in key:
            continue
        struct, field = key.split(".")
        cls = {"einet_layer_desc": _native.LayerDesc, "einet_plan_desc": _native.PlanDesc,
               "einet_sizes": _native.Sizes}[struct]
        assert getattr(cls, field).offset == int(value), key


def test_plan_create_rejects_bad_descriptors_on_host(native_lib):
    lib = native_lib
    h = ctypes.c_void_p()
    assert lib.einet_plan_create(None, 16, ctypes.byref(h)) == _native.ERR_USAGE
    assert "null" in _native.last_error()
    desc = _native.PlanDesc(d_vars=4, k=0, k_root=1, num_replicas=1, num_buffer_rows=2)
    assert lib.einet_plan_create(ctypes.byref(desc), 16, ctypes.byref(h)) == _native.ERR_USAGE
    desc = _native.PlanDesc(d_vars=4, k=2, k_root=1, num_replicas=1, num_buffer_rows=2,
                            family=7, n_leaf=1, n_layers=1)
    assert lib.einet_plan_create(ctypes.byref(desc), 16, ctypes.byref(h)) == _native.ERR_USAGE
    assert "family" in _native.last_error()
    assert lib.einet_mstep(None, None, None, None, 0.5, 1e-12, None, None) == _native.ERR_USAGE


def test_launch_counter_and_profile_query_without_gpu(native_lib):
    assert native_lib.einet_launch_count() >= 0
    assert _native.profile_read() == {}


def test_product_path_fails_loudly_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import numpy as np
    import paper_2004_06231_b200 as E
    rg = E.random_binary_tree(4, E.StructureConfig(depth=1, replicas=1, seed=0))
    with pytest.raises(_native.NativeUnavailable):
        E.build_model(rg, E.GaussianFamily(), k=2, seed=0, data=np.zeros((3, 4)))
