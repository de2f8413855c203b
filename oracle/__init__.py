"""ORACLE -- test infrastructure only (see ils_oracle.py header).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference leg
may import anything under oracle/.
"""
from . import index_stream, ils_oracle  # noqa: F401
