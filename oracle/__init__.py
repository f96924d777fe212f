"""CPU oracle for decimal -> nearest binary64 / binary32 (arXiv 2101.11408).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product path (``paper_2101_11408_b200``) never imports it, and it
never imports the product path: the two share no code, tables or constants.

The oracle is the *plain definition* of the result the paper's method reaches
(PAPER.md abstract L4-15: "parsing decimal numbers to the nearest binary
floating-point value"; ties to even, L42-46 and the notation table): the
decimal string is read as an exact rational and compared against binary64
candidates and their midpoints with Python's arbitrary-precision integers.
It uses no table T[q], no Algorithm 1 and no binary floating point anywhere in
its decision.

Modules
  records.py  record splitting (split variant) and record bounds (batch variant)
  lexer.py    record grammar (readings G7, G8, G10 in DESIGN.md)
  exact.py    exact correctly rounded conversion
  api.py      parse_batch / parse_split: whole-buffer entry points + pool runner

Parity pins: see tests/test_oracle_*.py (worked examples in tests/golden/,
round trip of 17-digit printing PAPER.md L55, brute force over tiny windows,
CPython float() as an independent correctly rounded library routine).
"""
from .exact import (STATUS_OK, STATUS_OVERFLOW, STATUS_UNDERFLOW, STATUS_INVALID,
                    STATUS_EMPTY, QNAN_BITS, round_decimal, QNAN32_BITS, round_decimal32)
from .lexer import lex_record, GRAMMAR_DEFAULT, GRAMMAR_HEX, GRAMMAR_JSON
from .api import parse_record, parse_batch, parse_split, split_records

__all__ = [
    "STATUS_OK", "STATUS_OVERFLOW", "STATUS_UNDERFLOW", "STATUS_INVALID", "STATUS_EMPTY",
    "QNAN_BITS", "round_decimal", "QNAN32_BITS", "round_decimal32", "lex_record",
    "GRAMMAR_DEFAULT", "GRAMMAR_HEX", "GRAMMAR_JSON", "parse_record", "parse_batch",
    "parse_split", "split_records",
]
