"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This package holds NONE of the method's arithmetic (no pyramid, patch distance, remap or blend):
only the input recipes of DESIGN.md §5 ("moving texture" videos shaped like the paper's workloads,
P:521 / BASELINE.json configs) and the small pin fixtures.
"""
from .video import *  # noqa: F401,F403
