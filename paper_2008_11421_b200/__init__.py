"""KARMA out-of-core data-parallel executor for B200 (arXiv 2008.11421).

The reference planner's plan.json drives ``libkrt.so`` (include/krt.h); see
DESIGN.md.  Importing the package does not load CUDA; ``_lib.lib()`` loads the
native library on first use and fails loudly when it has not been built.
"""
__version__ = "0.1.0"
