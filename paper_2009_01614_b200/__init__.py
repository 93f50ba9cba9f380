"""isax-b200: exact 1-NN Euclidean search over iSAX-summarised data series on one B200 (sm_100a).

The method is ParIS / ParIS+ / MESSI (arXiv 2009.01614). The product is libisax.so behind
include/isax.h. This package is its thin Python binding (`isax.Index`) plus the build script.

Importing `paper_2009_01614_b200.isax` loads libisax.so and fails loudly if it is missing.
This top-level import stays light, so the build can run before the library exists.
"""

__all__ = ["isax", "build"]
