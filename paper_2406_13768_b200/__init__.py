"""B200-native FastPersist: data-parallel checkpoint-write hot path.

Native library (csrc/, C-ABI in include/fastpersist.h) + this thin ctypes
binding. See DESIGN.md.
"""
from .fastpersist import (  # noqa: F401
    Checkpointer, Entry, FastPersistError, io_bench, lib, LIB_PATH, EXPORTS, StreamWriter, save,
)
