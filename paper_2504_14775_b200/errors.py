"""Error types raised across the host runtime.

Same names and hierarchy as the reference simulator
(`pkg/src/tokensim/errors.py:6-23`) so callers that catch `ConfigError` or
read `UnschedulableError.request_ids` keep working after the switch.
`NativeError` is new: it wraps a non-zero return code from the C-ABI
(`include/gllm.h`) together with `gllm_last_error()`.
"""

from __future__ import annotations


class SimError(Exception):
    """Root of every error this package raises on purpose."""


class ConfigError(SimError):
    """An invalid configuration value or combination."""


class TraceError(SimError):
    """A malformed request trace (JSONL) file."""


class UnschedulableError(SimError):
    """No forward progress is possible for the listed requests."""

    def __init__(self, message: str, request_ids: tuple[int, ...] = ()):
        super().__init__(message)
        self.request_ids = tuple(request_ids)


class NativeError(SimError):
    """A CUDA/C-ABI entry point returned an error code."""

    def __init__(self, func: str, code: int, detail: str):
        super().__init__(f"{func} failed with code {code}: {detail}")
        self.func = func
        self.code = code
        self.detail = detail
