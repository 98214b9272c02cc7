"""Exception types of the reference surface.

``ValidationError`` mirrors ``container.ValidationError`` (container.py:48-49)
and ``NumericError`` mirrors ``model.NumericError`` (model.py:24-25); both are
``ValueError`` subclasses exactly as in the reference, so callers that catch
the reference's exceptions catch these.
"""


class ValidationError(ValueError):
    """Invalid configuration, shape or position."""


class NumericError(ValueError):
    """Non-finite values reached a numeric kernel."""
