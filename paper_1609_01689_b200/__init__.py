"""B200-native (sm_100a) LOBPCG hot path of arXiv:1609.01689 behind the
reference's ci:: API (see ci.py, include/cieg.h)."""
from . import _lib  # noqa: F401

__all__ = ["ci"]
