"""Exception taxonomy of the reference toolchain (trafficsim/errors.py:4-36).

Kept name-for-name so code written against the reference's ``World`` catches
the same classes.  ``EngineError`` is new: a CUDA / native-library failure
surfaced through ``tsb_last_error()``; it derives from ``TrafficSimError``.
"""


class TrafficSimError(Exception):
    """Root of every error raised by this package."""


class InputError(TrafficSimError):
    """Bad user input (reference maps it to CLI exit code 2)."""


class ParseError(InputError):
    """Input document not structurally readable."""


class SchemaError(InputError):
    """Readable document that violates the expected schema."""


class BuildError(InputError):
    """Network compilation failure."""


class NoRouteError(TrafficSimError):
    """No lane path from origin to destination."""


class RecorderError(TrafficSimError):
    """Record sink failed mid-run."""


class EngineError(TrafficSimError):
    """The native B200 engine reported a failure (CUDA error, capacity)."""
