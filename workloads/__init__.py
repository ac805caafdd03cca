"""Synthetic workloads for the tests and bench.py.

Test/bench infrastructure, not product code: pure numpy/json, nothing here
imports the B200 package, so bench.py's reference arm builds the identical
tables and rows without loading libbbpe_b200.so.
"""
from . import tables, text  # noqa: F401
