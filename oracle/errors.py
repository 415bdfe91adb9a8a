"""Oracle-side error classes (test infrastructure only).

Mirror the reference hierarchy and exit codes (octowall/errors.py:4-41) so
the oracle can be compared on failure behaviour as well as on outputs.
"""


class OracleError(Exception):
    exit_code = 1


class InvalidParameter(OracleError):
    exit_code = 2


class ParseError(OracleError):
    exit_code = 3


class Capacity(OracleError):
    exit_code = 4
