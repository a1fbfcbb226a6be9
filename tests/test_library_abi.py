"""CPU checks of the C-ABI library (no GPU): it builds, loads, exports every symbol
declared in include/mhdp.h, and its host-only context rejects device calls loudly."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def mh():
    from paper_2104_14855_b200 import build_lib, mhdp
    build_lib.build()
    return mhdp


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "mhdp.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mhdp_[a-z_0-9]+)\s*\(", src)))


def test_every_declared_symbol_is_exported(mh):
    lib = mh.lib()
    decl = declared_symbols()
    assert len(decl) >= 25
    for name in decl:
        assert hasattr(lib, name), name
    assert sorted(mh.SYMBOLS) == decl


def test_host_only_context_rejects_device_calls(mh):
    ctx = mh.Context(-1)
    from paper_2104_14855_b200 import workloads
    cfg = workloads.CONFIGS["c1"]
    with pytest.raises(mh.MhdpError) as e:
        ctx.setup()
    assert e.value.status in (3, 5)
    st = ctx._L.mhdp_smooth(ctx.h, 0, 1, 1, 0, 0)
    assert st != 0


def test_invalid_arguments(mh):
    from paper_2104_14855_b200 import workloads
    ctx = mh.Context(-1)
    cfg = workloads.CONFIGS["c1"]
    w = workloads.advecting_potential(cfg, None)
    with pytest.raises(mh.MhdpError) as e:
        ctx.assemble(cfg, w, N=6, levels=3)        # 6 not divisible by 4
    assert e.value.status == 1
    bad = workloads.dataclasses.replace(cfg, Rem=0.0)
    with pytest.raises(mh.MhdpError):
        ctx.assemble(bad, w)
    # load_level validation: unsorted columns
    ctx.begin_levels(1, cfg)
    with pytest.raises(mh.MhdpError):
        ctx.load_level(0, np.array([0, 2]), np.array([0, 0]), np.array([1.0, 2.0]))


def test_missing_library_fails_loudly(mh, monkeypatch):
    """No CPU fallback: without libmhdp.so the binding raises (it never routes to the oracle
    or to PyTorch)."""
    monkeypatch.setattr(mh, "_lib", None)
    monkeypatch.setattr(mh, "LIB", os.path.join(ROOT, "build", "does_not_exist", "libmhdp.so"))
    with pytest.raises(OSError):
        mh.lib()
    with pytest.raises(OSError):
        mh.Context(-1)
