"""CPU oracle for the FastCHGNet training step — TEST INFRASTRUCTURE ONLY.

Plain, slow, fp64 implementation of what the hot path computes, written from
the paper (PAPER.md, arXiv 2412.20796) with the readings of SURVEY.md §8(c)
(listed in DESIGN.md "Readings").  Only `tests/`, `__graft_entry__.smoke()` and
`bench.py`'s `cpu_baseline` / `--impl reference` legs may import it.  It shares
no code with the CUDA path (`paper_2412_20796_b200/`) and never imports it.

Modules
  graph.py  — O1: periodic atom graph, bond graph, angle list, rev/swap maps
  model.py  — O2..O6, O8, O10: basis, embedding, interaction blocks, heads;
              gradients by torch autograd (exact reverse mode of the forward)
  train.py  — O7 loss, O9 Adam + LR (Eq. 14 × cosine), O11 balance sampler

Parity status per function is in DESIGN.md "Oracle pins"; functions without a
pin say "parity unpinned" in their docstring.
"""
