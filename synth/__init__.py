"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the CPU oracle.

Holds no arithmetic of the method (SURVEY.md Appendix B recipe only)."""
from .generator import *  # noqa: F401,F403
