"""Seeded synthetic inputs for the Zipage compression step.

This module is the ONE thing the oracle side (tests, bench cpu leg) and the CUDA
side share: it generates inputs and holds none of the method's arithmetic.
``philox`` is a counter-based generator (Philox4x32-10) with a bit-identical
device twin in ``csrc/zpc_gen.cu`` (built as ``libzpcgen.so``, separate from the
product library) so full-size pools can be generated in HBM while any sampled
request can be regenerated on the host. See DESIGN.md §Inputs for the recipe.
"""
from .philox import philox4x32  # noqa: F401
from .workloads import *  # noqa: F401,F403
