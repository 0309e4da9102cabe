"""Exception types of the path, matching the reference's (same names, same
base classes) so callers' ``except`` clauses keep working."""


class ParseError(ValueError):
    """relation.py:17-20."""

    def __init__(self, line_no: int, msg: str):
        super().__init__(f"line {line_no}: {msg}")
        self.line_no = line_no


class PlanError(ValueError):
    """optimizer.py:21-22."""


class MatrixOverflowError(OverflowError):
    """matmul/core.py:33-34."""


class StarResourceError(RuntimeError):
    """joinproject.py:28-29: heavy cross product too large; retry with a larger delta2."""
