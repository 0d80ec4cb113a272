"""CPU oracle package -- TEST INFRASTRUCTURE ONLY (see oracle/kvstream.py header).

Importable from tests/, __graft_entry__.smoke() and bench.py's cpu_baseline/reference legs only.
"""
from .kvstream import *  # noqa: F401,F403
from .kvstream import MappingError, RangeError, Setup, Piece, Cache  # noqa: F401
