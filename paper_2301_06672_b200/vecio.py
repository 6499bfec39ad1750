"""Record containers (.fvecs / .bvecs / .ivecs); they live in `datasets`
(reference datasets.py:60-137) -- re-exported here for older callers."""

from .datasets import read_bvecs, read_fvecs, read_ivecs, read_vectors, write_fvecs, write_ivecs  # noqa: F401
