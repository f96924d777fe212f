"""Record grammar for the oracle (test infrastructure only).

A plain byte-at-a-time reading of the record grammar fixed in DESIGN.md
("Record grammar"), which follows the paper's string-parsing steps
(PAPER.md section "Parsing the String", L158-185):
  * L167: the string is explicitly delimited; nothing outside it is read;
  * L168-170: no whitespace skipping (C locale, reading G8), optional '+'/'-';
  * L171: digits with an optional '.', at least one digit required;
  * L177-179: optional 'e'/'E' exponent with optional sign; an exponent
    character without digits makes the record INVALID (reading G7);
  * specials "inf", "infinity", "nan", ASCII case-insensitive (reading G10).

    record  := [sign] ( decimal [exp] | special ) terminator*
    decimal := digit+ [ '.' digit* ] | '.' digit+
    exp     := ('e'|'E') [sign] digit+
    terminator := '\\n' | '\\r' | ','

A record made only of terminator bytes (including the zero-length record) is
EMPTY.

Grammar options (readings H1-H3, J1):
  GRAMMAR_HEX  also accept C99 hexadecimal floats (PAPER.md "Hexadecimal
               Floating-Point Numbers", L1486-1497):
                 hexfloat := ('0x'|'0X') hexdigit* ['.' hexdigit*] [('p'|'P') [sign] digit+]
               with at least one hex digit; value = int(hexdigits, 16) * 2^(P - 4 * fraction
               nibbles) (the C99 reading of the hexadecimal point, H1; the
               exponent is optional as in strtod, H2).
  GRAMMAR_JSON only RFC 8259 numbers ("+1, 01, 1.e1" are invalid
               JSON; L171 leading zeros, empty integer or fraction parts):
                 ['-'] ('0' | [1-9] digit*) ['.' digit+] [('e'|'E') [sign] digit+]
               no specials, no '+', no hex (J1); terminators as above.

The decimal value is returned unreduced as (neg, digit string, Q) with
value int(digits) * 10^Q, Q = explicit exponent - number of fraction digits;
Q is an unbounded Python int (reading G9: the exact value is honoured).
Exponent digit strings of any length are converted exactly (exact.int_of_digits:
CPython's int(str) refuses more than 4300 digits, PAPER.md L179 sets no limit).
"""
from .exact import int_of_digits

_TERMINATORS = b"\n\r,"
_DIGITS = b"0123456789"
_HEXDIGITS = b"0123456789abcdefABCDEF"

GRAMMAR_DEFAULT = 0
GRAMMAR_HEX = 1
GRAMMAR_JSON = 2


def _lex_hex(rec, i, neg):
    """The hexadecimal float after its '0x' (i points past the 'x')."""
    n = len(rec)
    int_nib = []
    while i < n and rec[i] in _HEXDIGITS:
        int_nib.append(chr(rec[i]))
        i += 1
    frac_nib = []
    if i < n and rec[i] == ord("."):
        i += 1
        while i < n and rec[i] in _HEXDIGITS:
            frac_nib.append(chr(rec[i]))
            i += 1
    if not int_nib and not frac_nib:
        return ("invalid",)
    pexp = 0
    if i < n and rec[i] in b"pP":
        i += 1
        eneg = False
        if i < n and rec[i] in b"+-":
            eneg = rec[i] == ord("-")
            i += 1
        exp_digits = []
        while i < n and rec[i] in _DIGITS:
            exp_digits.append(chr(rec[i]))
            i += 1
        if not exp_digits:
            return ("invalid",)
        pexp = int_of_digits("".join(exp_digits))
        if eneg:
            pexp = -pexp
    while i < n:
        if rec[i] not in _TERMINATORS:
            return ("invalid",)
        i += 1
    return ("hex", neg, "".join(int_nib) + "".join(frac_nib), pexp - 4 * len(frac_nib))


def lex_record(rec, grammar=GRAMMAR_DEFAULT):
    """Lex one record (bytes) under the grammar option (GRAMMAR_*).

    Returns one of
      ("empty",)            only terminator bytes (or zero length)
      ("invalid",)          anything the grammar rejects
      ("inf", neg) / ("nan", neg)
      ("num", neg, digits: str, Q: int)
      ("hex", neg, hexdigits: str, E2: int)   value int(hexdigits, 16) * 2^E2
    """
    json = grammar & GRAMMAR_JSON
    n = len(rec)
    if all(b in _TERMINATORS for b in rec):
        return ("empty",)
    i = 0
    neg = False
    if rec[i] in (b"-" if json else b"+-"):
        neg = rec[i] == ord("-")
        i += 1
    # specials: whole remaining body (before terminators) compared case-insensitively
    j = n
    while j > i and rec[j - 1] in _TERMINATORS:
        j -= 1
    body = bytes(rec[i:j]).lower()
    if not json:
        if body in (b"inf", b"infinity"):
            return ("inf", neg)
        if body == b"nan":
            return ("nan", neg)
    if (grammar & GRAMMAR_HEX) and not json and body[:2] == b"0x":
        return _lex_hex(rec, i + 2, neg)
    # decimal part
    int_digits = []
    while i < n and rec[i] in _DIGITS:
        int_digits.append(chr(rec[i]))
        i += 1
    frac_digits = []
    dot = False
    if i < n and rec[i] == ord("."):
        dot = True
        i += 1
        while i < n and rec[i] in _DIGITS:
            frac_digits.append(chr(rec[i]))
            i += 1
    if not int_digits and not frac_digits:
        return ("invalid",)
    if json:
        # int := '0' | [1-9] digit*;  frac := '.' digit+
        if not int_digits or (len(int_digits) > 1 and int_digits[0] == "0"):
            return ("invalid",)
        if dot and not frac_digits:
            return ("invalid",)
    exp = 0
    if i < n and rec[i] in b"eE":
        i += 1
        eneg = False
        if i < n and rec[i] in b"+-":
            eneg = rec[i] == ord("-")
            i += 1
        exp_digits = []
        while i < n and rec[i] in _DIGITS:
            exp_digits.append(chr(rec[i]))
            i += 1
        if not exp_digits:
            return ("invalid",)
        exp = int_of_digits("".join(exp_digits))
        if eneg:
            exp = -exp
    # the rest of the record may only hold terminators
    while i < n:
        if rec[i] not in _TERMINATORS:
            return ("invalid",)
        i += 1
    digits = "".join(int_digits) + "".join(frac_digits)
    return ("num", neg, digits, exp - len(frac_digits))
