"""CPU-side checks of the C-ABI library (no GPU calls): it was built for
sm_100a, it loads, it exports every symbol include/chg.h declares, and the
host-only sampler (chg_balance) matches the oracle's."""
import os
import re
import shutil
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2412_20796_b200 import chg
    if not os.path.exists(chg.LIB_PATH):
        import __graft_entry__
        __graft_entry__.build()
    return chg.load()


def _header_symbols():
    txt = open(os.path.join(ROOT, "include", "chg.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(chg_[a-z0-9_]+)\s*\(", txt)))


def test_exports_every_declared_symbol(lib):
    from paper_2412_20796_b200 import chg
    syms = _header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(chg.SYMBOLS) == syms


def test_built_for_sm100a():
    from paper_2412_20796_b200 import chg
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not found")
    out = subprocess.run(["cuobjdump", "--list-elf", chg.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_balance_matches_oracle(lib):
    from oracle.train import balance_assign
    from paper_2412_20796_b200 import chg
    rng = np.random.default_rng(0)
    for W in (1, 2, 3, 8):
        loads = rng.integers(1, 50, size=101)          # many ties
        ref = balance_assign(list(loads), W)
        got = chg.balance(loads, W)
        for r, ids in enumerate(ref):
            assert sorted(np.nonzero(got == r)[0].tolist()) == sorted(ids)
    with pytest.raises(chg.ChgError):
        chg.balance([1, 2], 0)


def test_no_cpu_fallback_without_library(tmp_path):
    """The binding refuses to run without the CUDA library (no CPU path)."""
    from paper_2412_20796_b200 import chg
    old = chg._lib
    try:
        chg._lib = None
        with pytest.raises(ImportError):
            chg.load(str(tmp_path / "missing.so"))
    finally:
        chg._lib = old
