"""Host-side checks of the C-ABI library (no GPU needed): it loads, exports
every symbol include/mpjsvd.h declares, and fails cleanly without a GPU."""
import ctypes as C
import os
import re

import pytest

import paper_2209_04626_b200 as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "mpjsvd.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mpjsvd_[a-z0-9_]+)\s*\(", src)))


def test_library_builds_and_loads():
    from paper_2209_04626_b200 import build
    build.build()
    assert os.path.exists(mp.LIB_PATH)
    mp.lib()


def test_exports_every_header_symbol():
    L = C.CDLL(mp.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 14
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(mp.EXPORTS)


def test_strerror_and_defaults():
    assert mp.strerror(0) == "ok"
    for code in (1, -1, -2, -3, -4, -5, -6, -7, 12345):
        assert isinstance(mp.strerror(code), str) and mp.strerror(code)
    o = mp.default_options()
    assert o.block_cols == 32 and o.tol_mult64 == 4.0 and o.inner_tol_div == 8
    assert o.max_sweeps32 == 20 and o.max_sweeps64 == 30 and o.x_from_lq == 1
    assert mp.lib().mpjsvd_version() == 150
    assert o.virtual_shards == 1 and o.split_rows == 0


def test_struct_layouts_match_header(tmp_path):
    """ctypes mirrors of mpjsvd_options / mpjsvd_stats agree with the C
    compiler's layout of include/mpjsvd.h (size and every field offset)."""
    import subprocess
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "mpjsvd.h"', 'int main(void){']
    for cname, py in (("mpjsvd_options", mp.Options), ("mpjsvd_stats", mp.Stats)):
        lines.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for f, _ in py._fields_:
            lines.append(f'printf("{cname}.{f} %zu\\n", offsetof({cname}, {f}));')
    lines.append("return 0;}")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    out = dict(l.split() for l in subprocess.check_output([str(exe)]).decode().splitlines())
    for cname, py in (("mpjsvd_options", mp.Options), ("mpjsvd_stats", mp.Stats)):
        assert int(out[cname]) == C.sizeof(py), cname
        for f, _ in py._fields_:
            assert int(out[f"{cname}.{f}"]) == getattr(py, f).offset, f


def test_invalid_arguments_rejected_without_gpu():
    L = mp.lib()
    # NULL handle / NULL pointers are rejected before any CUDA call
    assert L.mpjsvd_factor(None, None, 4, 4, 4, None, 4, None, None, 4, None) == -1
    assert L.mpjsvd_destroy(None) == 0
    o = mp.default_options(block_cols=7)
    h = C.c_void_p()
    assert L.mpjsvd_create(C.byref(h), C.byref(o)) == -7
    o = mp.default_options(num_gpus=2)
    assert L.mpjsvd_create(C.byref(h), C.byref(o)) == -7


def test_create_without_gpu_fails_cleanly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = C.c_void_p()
    rc = mp.lib().mpjsvd_create(C.byref(h), None)
    assert rc < 0 and not h.value


def test_comm_entry_points_without_gpu():
    """NCCL is dlopen'd lazily: the unique id is produced (or MPJSVD_ERR_NCCL is
    returned cleanly) without a GPU, and bad arguments are rejected."""
    L = mp.lib()
    buf = C.create_string_buffer(mp.COMM_ID_BYTES)
    rc = L.mpjsvd_comm_unique_id(buf)
    assert rc in (0, -5)
    assert L.mpjsvd_comm_unique_id(None) == -1
    assert L.mpjsvd_comm_init(None, 0, 1, buf) == -1
    o = mp.default_options(virtual_shards=0)
    h = C.c_void_p()
    assert L.mpjsvd_create(C.byref(h), C.byref(o)) == -1
