"""CADET (arXiv 2602.11410) hot path on B200: packed, session-masked, self-gated timestamp-RoPE
attention + context-conditioned towers, as hand-written sm_100a CUDA behind the libcadet C ABI
(include/cadet.h).  `ops` is the torch-facing binding; `_lib` the raw ctypes one."""
from . import _lib  # noqa: F401

__all__ = ["_lib", "ops"]
