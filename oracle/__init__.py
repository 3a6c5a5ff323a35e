"""CPU oracle for arxiv 1711.00244 ("inference from compressed models under
memory constraints").  TEST INFRASTRUCTURE ONLY.

This package is a plain, slow, obviously-correct CPU implementation of what the
hot path computes, written from PAPER.md (cited as P:Lnnn) with the readings of
SURVEY.md §8(c) (cited as C-nn, listed in DESIGN.md).  Floating point is fp64
unless the paper fixes the precision (the stored codebook is fp32).

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline /
`--impl reference` legs may import, call or execute anything under `oracle/`.
The product (`paper_1711_00244_b200/`) never imports it, and it never imports
the product.  It shares code with the product only through `synth/`, which
holds the seeded input generators and none of the method's arithmetic.

Modules, in pipeline order (Fig. 1a-1e):
  prune      magnitude pruning to an exact kept count            (C-10)
  quantize   r-bit codebook, linear init, nearest centre         (C-04/05/07)
  relindex   k-bit relative column index with padding zeros      (C-01/02/03)
  huffman    Huffman build / canonical codes / encode / decode   (C-14..17)
  cdni       CDNI container serialise / parse
  compress   the whole pipeline: dense W -> CDNI layer
  decode     Algorithm 1 lines 4-8: row-wise decode
  infer      FC (Eq. 1-2), CONV via im2col, LRN, max-pool
  planner    §6 dynamic program, fixed-batch baseline, brute force

Pins for every function live in tests/test_oracle_*.py (run with -m "not gpu").
Parity unpinned (oracle-defined, no independent pin): LRN constants (C-20).
"""
