"""Exception taxonomy of the drop-in API (mirrors moesim/errors.py:8-31 by name).

ConfigError      invalid parameters, raised before any device work (C-ABI MOE_INVALID_CONFIG)
TraceError       trace / event-log file problems
  TraceParseError       malformed line (carries the 1-based line number)
  TraceValidationError  data-model invariant violated
Non-finite gate logits raise the builtin FloatingPointError (toymoe.py:109-110).
"""

from __future__ import annotations


class MoesimError(Exception):
    """Root of the package's own exceptions."""


class ConfigError(MoesimError):
    pass


class TraceError(MoesimError):
    pass


class TraceParseError(TraceError):
    def __init__(self, message: str, line: int | None = None):
        self.line = line
        super().__init__(message if line is None else f"line {line}: {message}")


class TraceValidationError(TraceError):
    pass
