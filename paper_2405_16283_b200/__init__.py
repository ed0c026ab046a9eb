"""B200-native executor for Turnip memgraphs (arXiv 2405.16283).

`memplan` mirrors the reference memplan Python API (bit-exact planner,
virtual-time dispatcher); `executor` runs memgraphs on B200 GPUs.
"""
from ._lib import MemplanError  # noqa: F401

__version__ = "0.1"
