"""kascade.errors (errors.py): the exception taxonomy."""
from ..exceptions import (FormatError, InvalidArgumentError, InvalidPlanError, KascadeError, NumericError,
                          UndefinedScoreError, UnsupportedOperationError)

__all__ = ["FormatError", "InvalidArgumentError", "InvalidPlanError", "KascadeError", "NumericError",
           "UndefinedScoreError", "UnsupportedOperationError"]
