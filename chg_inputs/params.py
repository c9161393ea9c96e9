"""Seeded parameter blobs (initialisation recipe: SURVEY.md §8(c) Q29).

The caller passes its OWN layout (list of (name, shape)); this module does not
define the model's layout, so the oracle and the CUDA library each keep their
own table and a test checks that they agree.

Recipe: 2-D weights [in,out] ~ U(±1/sqrt(in)); biases and LN offsets 0; LN
gains 1; radial frequencies f_n = nπ (n = 1..K).  Names decide the kind:
  *.freq -> nπ;  *.g (LayerNorm gain) -> 1;  1-D others -> 0;  2-D -> uniform.
"""
from __future__ import annotations

import math
from typing import Sequence, Tuple

import numpy as np


def init_flat_params(layout: Sequence[Tuple[str, Tuple[int, ...]]], seed: int = 0,
                     bias_scale: float = 0.0) -> np.ndarray:
    """Flat float64 parameter vector in `layout` order.  `bias_scale` > 0 draws
    biases and LN offsets from U(±bias_scale) and LN gains from 1+U(±bias_scale)
    instead of 0/1 (used by tests so that every parameter is exercised)."""
    rng = np.random.default_rng(seed)
    out = []
    for name, shape in layout:
        n = int(np.prod(shape))
        leaf = name.rsplit(".", 1)[-1]
        if leaf == "freq":
            v = np.arange(1, n + 1, dtype=np.float64) * math.pi
        elif len(shape) == 2:
            bound = 1.0 / math.sqrt(shape[0])
            v = rng.uniform(-bound, bound, size=n)
        elif leaf == "g":
            v = np.ones(n) + (rng.uniform(-bias_scale, bias_scale, size=n) if bias_scale else 0.0)
        else:
            v = rng.uniform(-bias_scale, bias_scale, size=n) if bias_scale else np.zeros(n)
        out.append(np.asarray(v, dtype=np.float64).reshape(-1))
    return np.concatenate(out)
