"""fp64 CPU oracle (test infrastructure only; see compact_attention.py header)."""
from .compact_attention import *  # noqa: F401,F403
