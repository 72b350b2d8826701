"""Exceptions of the drop-in API, named and layered as in the reference.

memory.py:44-57 (SimMemoryError, OutOfSimMemory, WildAccess, AttachOutsideArena) and
harness.py:46-51 (VerificationFailed, SchemeError).  The native library reports failures as
CF_E_* codes (include/chainforge_b200.h); ``_native.check`` maps them onto these classes.
"""


class SimMemoryError(Exception):
    """Base class for memory-space faults (kept under the reference's name)."""


class OutOfSimMemory(SimMemoryError):
    pass


class WildAccess(SimMemoryError):
    """Access to an address outside any live allocation of a space."""


class AttachOutsideArena(SimMemoryError):
    """A pointer fix-up targeted memory that is not part of the arena."""


class VerificationFailed(Exception):
    pass


class SchemeError(ValueError):
    pass


class NativeUnavailable(RuntimeError):
    """The CUDA extension is missing or no GPU is visible: the product path never falls back."""
