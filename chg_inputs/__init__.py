"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NO arithmetic of the method (no graph, basis, model, loss or
optimizer code).  It only draws random crystals, labels and parameter blobs
from documented recipes.
Both `oracle/` and the CUDA path's tests/bench consume it; neither imports the
other.
"""
from .structures import (  # noqa: F401
    Batch,
    si_diamond,
    simple_cubic,
    dimer,
    mptrj_like_batch,
    skewed_oxide_batch,
    lifepo4_like_cell,
    concat_batches,
    split_batch,
    make_config_batch,
    random_rotation,
)
from .params import init_flat_params  # noqa: F401
from .lj import lj_dataset, lj_labels  # noqa: F401
