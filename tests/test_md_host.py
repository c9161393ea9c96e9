"""Host-side checks of the MD loop's units and initial conditions."""
import os
import re
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2412_20796_b200.md import EV_PER_AMU_A2_FS2, KB_EV, maxwell_boltzmann  # noqa: E402


def test_unit_constants_from_si():
    amu, ev = 1.66053906660e-27, 1.602176634e-19          # kg, J (CODATA 2018)
    assert abs(EV_PER_AMU_A2_FS2 - amu * 1e-20 / 1e-30 / ev) < 1e-6
    assert abs(KB_EV - 1.380649e-23 / ev) < 1e-12
    # the kernel's acceleration unit (eV/Å/amu -> Å/fs²) is the inverse of the same factor
    src = open(os.path.join(ROOT, "paper_2412_20796_b200", "csrc", "md.cu")).read()
    acc = float(re.search(r"ACC_UNIT = ([0-9.eE+-]+);", src).group(1))
    assert abs(acc * EV_PER_AMU_A2_FS2 - 1.0) < 1e-9


def test_maxwell_boltzmann_temperature_and_momentum():
    m = np.random.default_rng(0).uniform(1.0, 200.0, 20000)
    v = maxwell_boltzmann(m, 300.0, seed=3)
    assert np.abs((m[:, None] * v).sum(0)).max() < 1e-9
    ke = 0.5 * (m[:, None] * v * v).sum() * EV_PER_AMU_A2_FS2
    t = 2.0 * ke / (3.0 * len(m) * KB_EV)
    assert abs(t - 300.0) < 6.0


def test_captured_md_needs_a_skin_graph():
    """NVE(captured=True) replays a fixed-topology step: without a skin (lists rebuilt every step)
    there is nothing to capture — refused before any device work."""
    import pytest
    from paper_2412_20796_b200.md import NVE

    class _Ctx:
        device = 0

    with pytest.raises(ValueError):
        NVE(_Ctx(), None, [0, 1], np.zeros((1, 3)), np.eye(3)[None], [14], [28.0], captured=True, skin=0.0)
