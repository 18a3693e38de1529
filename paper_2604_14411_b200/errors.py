"""Error classes of the partitioner.

The names and the inheritance tree are the reference's public contract
(errors.py:4-27 of dhgpart); ``STATUS`` maps libdhgp status codes
(include/dhgp.h) onto them.
"""


class DhgError(Exception):
    """Root of every error raised by this package."""


class DhgParseError(DhgError):
    """Input text (hypergraph or partition file) could not be parsed;
    ``line`` is the 1-based line number when known."""

    def __init__(self, message, line=None):
        self.line = line
        super().__init__(message if line is None else f"line {line}: {message}")


class InfeasibleError(DhgError):
    """No assignment can meet the size / distinct-inbound limits."""


class OracleSizeError(DhgError):
    """Exhaustive search requested on an instance that is too large."""


class MatchingInvariantError(DhgError):
    """The candidate pseudo-forest had a cycle longer than two."""


STATUS = {
    1: InfeasibleError,
    2: DhgError,
    3: MatchingInvariantError,
    4: DhgError,
}
