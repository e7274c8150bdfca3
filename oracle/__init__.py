"""DHEN fp64 CPU oracle — test infrastructure only (see dhen_oracle.py header)."""
from .dhen_oracle import *  # noqa: F401,F403
