"""CPU checks of the boundary: libgear.so builds, loads and exports every
entry point include/gear.h declares, with the binding's names; the oracle and
the product share no code.  No compute calls (no GPU here)."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "gear.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return set(re.findall(r"^\s*(?:gear_status|const char\*|uint64_t)\s+(gear_\w+)\s*\(", src, flags=re.M))


def test_header_declares_hot_path_calls():
    names = _declared()
    for n in ("gear_table_create", "gear_insert", "gear_update_priorities", "gear_sample",
              "gear_collect", "gear_table_destroy", "gear_comm_create", "gear_get_unique_id"):
        assert n in names


def test_library_exports_every_declared_symbol():
    import paper_2310_05205_b200 as gear
    from paper_2310_05205_b200 import build
    build.build()
    lib = ctypes.CDLL(gear.LIB_PATH)
    names = _declared()
    for n in names:
        assert hasattr(lib, n), f"libgear.so does not export {n}"
    # the binding wraps every declared entry point under the same name
    assert names == set(gear.SIGNATURES)
    for n in names - {"gear_last_error", "gear_version"}:
        assert callable(getattr(gear, n)), n
    assert gear.load().gear_version().startswith(b"gear-b200")
    assert gear.load().gear_last_error() == b""


def test_kernels_are_sm100a():
    """The fat binary carries sm_100a SASS (cuobjdump lists the arch)."""
    import subprocess
    import paper_2310_05205_b200 as gear
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", gear.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _imports_and_includes(path):
    out = []
    for line in open(path):
        m = re.match(r"\s*#\s*include\s*[<\"]([^>\"]+)[>\"]", line)
        if m:
            out.append(m.group(1))
        m = re.match(r"\s*(?:from|import)\s+([\w.]+)", line)
        if m and path.endswith(".py"):
            out.append(m.group(1))
    return out


def test_oracle_and_product_share_no_code():
    """Neither side includes, imports or links the other."""
    prod = os.path.join(ROOT, "paper_2310_05205_b200")
    for dp, _, fs in os.walk(prod):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                for dep in _imports_and_includes(os.path.join(dp, f)):
                    assert "oracle" not in dep, (f, dep)
    odir = os.path.join(ROOT, "oracle")
    for f in os.listdir(odir):
        if f.endswith((".c", ".h", ".py")):
            for dep in _imports_and_includes(os.path.join(odir, f)):
                assert "paper_2310_05205_b200" not in dep and "gear.h" != dep \
                    and "synth" not in dep, (f, dep)


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    """No CPU fallback: without libgear.so every call raises instead of
    computing anything on the host."""
    import pytest
    import paper_2310_05205_b200 as gear
    monkeypatch.setattr(gear, "_lib", None)
    monkeypatch.setattr(gear, "LIB_PATH", str(tmp_path / "libgear.so"))
    with pytest.raises(ImportError, match="no CPU fallback"):
        gear.load()
    with pytest.raises(ImportError):
        gear.gear_sample(1, gear.GEAR_PRIORITIZED, 4, 1, 0.4, 0, None, None, None, 0)


def test_binding_checks_dtypes_and_sizes():
    """The ctypes binding refuses tensors whose dtype or size would make a
    kernel read or write past the buffer: checked before the
    library is called, so no table or GPU is needed."""
    import numpy as np
    import pytest
    import torch
    import paper_2310_05205_b200 as G
    i64 = torch.zeros(8, dtype=torch.int64)
    i32 = torch.zeros(8, dtype=torch.int32)
    f32 = torch.zeros(8, dtype=torch.float32)
    f64 = torch.zeros(8, dtype=torch.float64)
    with pytest.raises(TypeError, match="out_idx"):
        G.gear_sample(0, G.GEAR_UNIFORM, 8, 1, 0.0, i32)
    with pytest.raises(TypeError, match="out_w"):
        G.gear_sample(0, G.GEAR_UNIFORM, 8, 1, 0.0, i64, f64)
    with pytest.raises(TypeError, match="out_p"):
        G.gear_sample(0, G.GEAR_UNIFORM, 8, 1, 0.0, i64, f32, f32)
    with pytest.raises(TypeError, match="out_gen"):
        G.gear_sample(0, G.GEAR_UNIFORM, 8, 1, 0.0, i64, f32, f64, f32)
    with pytest.raises(ValueError, match="elements"):
        G.gear_sample(0, G.GEAR_UNIFORM, 9, 1, 0.0, i64)
    with pytest.raises(TypeError, match="prio"):
        G.gear_update_priorities(0, 8, i64, f32, G.GEAR_F64)
    with pytest.raises(TypeError, match="idx"):
        G.gear_update_priorities(0, 8, i32, f64, G.GEAR_F64)
    with pytest.raises(TypeError, match="gen"):
        G.gear_update_priorities(0, 8, i64, f64, G.GEAR_F64, gen=i64)
    with pytest.raises(TypeError, match="prio"):
        G.gear_commit(0, 0, 8, i64, f32)
    with pytest.raises(TypeError, match="out_idx"):
        G.gear_allocate(0, 0, 8, np.zeros(8, np.int32))
    with pytest.raises(TypeError, match="float32 or float64"):
        G.Table.update_priorities(type("T", (), {"handle": 0})(), i64, torch.zeros(8, dtype=torch.bfloat16))
