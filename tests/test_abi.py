"""CPU: the C-ABI library loads, exports every symbol include/fastleg_b200.h
declares, refuses to compute without a device (no CPU fallback), validates
arguments in the reference's order, and its host input generators reproduce
random.hpp bit-for-bit."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT
import paper_1505_00354_b200 as fl
from paper_1505_00354_b200 import _lib


def header_symbols():
    src = open(os.path.join(ROOT, "include", "fastleg_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fl_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_header_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(_lib.EXPORTS) == syms


def test_library_is_sm100a_cubin():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_validation_before_device_use():
    with pytest.raises(fl.InvalidArgument, match="size must be positive"):
        fl.legendre_nodes_weights(0)
    with pytest.raises(fl.InvalidArgument, match="dct_iii: empty input"):
        fl.dct_iii(np.zeros(0), fl.GridKind.cheb1)
    with pytest.raises(fl.InvalidArgument, match="dst_iii_transpose: empty input"):
        fl.dst_iii_transpose(np.zeros(0), fl.GridKind.chebstar)
    with pytest.raises(fl.InvalidArgument):
        fl.min_taylor_terms(fl.GridKind.cheb1, 0.0)
    with pytest.raises(fl.DomainError):
        fl.min_taylor_terms(fl.GridKind.cheb1, 1e-36)
    plan = fl.TaylorPlan(8, fl.GridKind.chebstar, 2.0 ** -52, 9,
                         fl.ReferenceGrid(8, fl.GridKind.chebstar, np.zeros(8), np.zeros(8)))
    with pytest.raises(fl.InvalidArgument, match="input size does not match plan"):
        fl.ndct_apply(plan, np.zeros(9))
    with pytest.raises(fl.InvalidArgument, match="expected Legendre"):
        fl.leg2cheb_apply(fl.chebyshev_coefficients(np.zeros(4)))
    with pytest.raises(fl.InvalidArgument, match="Lambda cache smaller"):
        _lib.check(_lib.LIB.fl_leg2cheb(0, 8, ctypes.c_void_p(np.zeros(4).ctypes.data), 4,
                                        ctypes.c_void_p(np.zeros(8).ctypes.data),
                                        ctypes.c_void_p(np.zeros(8).ctypes.data), 1, 8, None))


@pytest.mark.skipif(fl.device_available(), reason="a CUDA device is present")
def test_no_cpu_fallback():
    with pytest.raises(fl.FastlegCudaError, match="no CPU fallback"):
        fl.legendre_nodes_weights(8)
    with pytest.raises(fl.FastlegCudaError):
        fl.dct_iii(np.ones(8), fl.GridKind.cheb1)
    with pytest.raises(fl.FastlegCudaError):
        fl.TransformConfig(16)


def test_host_generators_match_random_hpp():
    from oracle import ORACLE, uniform_pm1
    for seed, decay in ((1, 0.5), (3, 1.0), (1000, 0.0)):
        assert np.array_equal(fl.random_decaying(257, decay, seed), ORACLE.random_decaying(257, decay, seed))
    b = fl.random_uniform_pm1(64, 4000, batch=3)
    for j in range(3):
        assert np.array_equal(b[j], uniform_pm1(64, 4000 + j))
    b = fl.random_decaying(33, 0.0, 1000, batch=4, threads=2)
    assert np.array_equal(b[2], ORACLE.random_decaying(33, 0.0, 1002))


def test_entry_imports_without_library():
    """A fresh checkout has no library yet: __graft_entry__ (whose build() makes
    it) must import, while the package itself must refuse loudly."""
    import subprocess
    import sys
    env = dict(os.environ, FLB_LIB_PATH=os.path.join(ROOT, "no_such_lib.so"))
    ok = subprocess.run([sys.executable, "-c", "import __graft_entry__ as g; assert callable(g.build)"],
                        cwd=ROOT, env=env, capture_output=True, text=True)
    assert ok.returncode == 0, ok.stderr
    bad = subprocess.run([sys.executable, "-c", "import paper_1505_00354_b200"],
                         cwd=ROOT, env=env, capture_output=True, text=True)
    assert bad.returncode != 0 and "no CPU fallback" in bad.stderr
