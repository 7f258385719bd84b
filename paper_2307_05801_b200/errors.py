"""Error hierarchy of the drop-in API.

Names, bases and meanings follow the reference package (pkg/src/ctproj/errors.py),
so ``except ctproj.errors.SpecMismatchError`` style handlers keep working
after switching.  Two classes are new and concern the native layer only:
``NativeLibraryError`` (the CUDA extension is missing or failed to load --
there is deliberately no CPU fallback) and ``CudaRuntimeError`` (a status
code from the C-ABI, include/ctproj_b200.h).
"""


class CtprojError(Exception):
    """Root of every error raised by this package (errors.py:4)."""


# -- configuration documents (geometry.parse_config) ------------------------
class ConfigError(CtprojError, ValueError):
    """A configuration document is invalid (errors.py:8)."""


class MissingKeyError(ConfigError):
    """A required configuration key is absent."""


class UnknownKeyError(ConfigError):
    """A configuration key is not recognised (typos fail loudly)."""


class InvalidValueError(ConfigError):
    """A configuration value has the wrong type or range."""


class ConflictingKeysError(ConfigError):
    """Two mutually exclusive keys were both given."""


# -- operator contracts ------------------------------------------------------
class UnsupportedGeometryError(CtprojError, ValueError):
    """The operation is not defined for this geometry kind (errors.py:28)."""


class SpecMismatchError(CtprojError, ValueError):
    """An array's shape/dtype/finiteness disagrees with the spec (errors.py:32)."""


class NonFiniteDataError(CtprojError, ValueError):
    """Input values contain NaN or infinity."""


class SizeMismatchError(CtprojError, ValueError):
    """An element count disagrees with the declared shape."""


class MalformedHeaderError(CtprojError, ValueError):
    """A raw-array header cannot be parsed."""


class LengthMismatchError(CtprojError, ValueError):
    """A per-view mask has the wrong length."""


class IndexOutOfRangeError(CtprojError, IndexError):
    """A (view, row, col) sample index is outside the detector."""


class DivergenceDetectedError(CtprojError, RuntimeError):
    """An iterative solve diverged."""


# -- native layer (new) ------------------------------------------------------
class NativeLibraryError(CtprojError, RuntimeError):
    """libctproj_b200.so is missing, stale or cannot be loaded.  Raised instead
    of silently falling back to any CPU path."""


class CudaRuntimeError(CtprojError, RuntimeError):
    """The C-ABI returned a CUDA / out-of-memory / workspace status."""
