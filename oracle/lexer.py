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
EMPTY.  The decimal value is returned unreduced as (neg, digit string, Q) with
value int(digits) * 10^Q, Q = explicit exponent - number of fraction digits;
Q is an unbounded Python int (reading G9: the exact value is honoured).
"""

_TERMINATORS = b"\n\r,"
_DIGITS = b"0123456789"


def lex_record(rec):
    """Lex one record (bytes).

    Returns one of
      ("empty",)            only terminator bytes (or zero length)
      ("invalid",)          anything the grammar rejects
      ("inf", neg) / ("nan", neg)
      ("num", neg, digits: str, Q: int)
    """
    n = len(rec)
    if all(b in _TERMINATORS for b in rec):
        return ("empty",)
    i = 0
    neg = False
    if rec[i] in b"+-":
        neg = rec[i] == ord("-")
        i += 1
    # specials: whole remaining body (before terminators) compared case-insensitively
    j = n
    while j > i and rec[j - 1] in _TERMINATORS:
        j -= 1
    body = bytes(rec[i:j]).lower()
    if body in (b"inf", b"infinity"):
        return ("inf", neg)
    if body == b"nan":
        return ("nan", neg)
    # decimal part
    int_digits = []
    while i < n and rec[i] in _DIGITS:
        int_digits.append(chr(rec[i]))
        i += 1
    frac_digits = []
    if i < n and rec[i] == ord("."):
        i += 1
        while i < n and rec[i] in _DIGITS:
            frac_digits.append(chr(rec[i]))
            i += 1
    if not int_digits and not frac_digits:
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
        exp = int("".join(exp_digits))
        if eneg:
            exp = -exp
    # the rest of the record may only hold terminators
    while i < n:
        if rec[i] not in _TERMINATORS:
            return ("invalid",)
        i += 1
    digits = "".join(int_digits) + "".join(frac_digits)
    return ("num", neg, digits, exp - len(frac_digits))
