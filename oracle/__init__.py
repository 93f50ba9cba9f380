"""Oracle for the iSAX exact 1-NN hot path. It is TEST INFRASTRUCTURE only.

This package is a plain, slow CPU implementation of what the paper's method computes
(arXiv 2009.01614, §Preliminaries and §Proposed Solution).

Only these callers may import, link or run it:
* `tests/`;
* `__graft_entry__.smoke()`;
* the `cpu_baseline` leg and `--impl reference` arm of `bench.py`.

The product path (`paper_2009_01614_b200/`) never imports it. The two share no code, headers,
tables or constant generators. The only code both sides use is the seeded input generator
in `datagen/`, and that holds none of the method's arithmetic.

Modules:
* `breakpoints`: the N(0,1) quantile table, correctly rounded, computed with mpmath.
* `ref`: numpy / pure-Python definitions (z-norm, PAA, SAX, key order, LB, ED, exact 1-NN,
  ParIS-style index search).
* `clib`: a ctypes wrapper for `oracle.c` (plain C + OpenMP), the same definitions for
  large inputs.

"parity unpinned" functions: none among the definitions. Candidate counts and pruning
ratios are reported, not pinned.
"""
