"""Exception types of the drop-in API (reference: errors.py:9-46).

Precondition violations raise plain ``ValueError``; ``ConfigError`` marks an
invalid configuration (bad pool shape, bad estimator config, bad snapshot).
The trace errors exist so callers that catch them keep working.
"""


class ConfigError(ValueError):
    """A run configuration is invalid (errors.py:9-10)."""


class TraceError(ValueError):
    """Base class for problems in a trace file (errors.py:13-14)."""


def _where(line, byte):
    parts = []
    if line is not None:
        parts.append(f"line {line}")
    if byte is not None:
        parts.append(f"byte {byte}")
    return f" ({', '.join(parts)})" if parts else ""


class TraceParseError(TraceError):
    """A record could not be decoded (errors.py:17-30)."""

    def __init__(self, message: str, *, line=None, byte=None):
        super().__init__(message + _where(line, byte))
        self.line = line
        self.byte = byte


class TraceOrderError(TraceError):
    """Timestamps in a trace went backwards (errors.py:33-46)."""

    def __init__(self, message: str, *, line=None, byte=None):
        super().__init__(message + _where(line, byte))
        self.line = line
        self.byte = byte
