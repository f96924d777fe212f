# Mutation check for the binary64 oracle pins (run by hand: python tests/mutate_oracle_f64.py).
# Each listed change to oracle/ must make the -m "not gpu" oracle pins fail
# (tests/test_oracle_pins.py, test_oracle_long_pins.py, test_oracle_grammar_pins.py).
# Exit status 1 if any mutation survives.  Mutations of the binary64 part of
# exact.py are applied before "def round_decimal32" only.
import subprocess
import sys

PINS = ["tests/test_oracle_pins.py", "tests/test_oracle_long_pins.py", "tests/test_oracle_grammar_pins.py"]

# (file, original, mutated, region): region "f64" = the part of exact.py before round_decimal32
MUTS = [
    ("oracle/exact.py", "return sign | ((e + 1075) << 52) | (m - _TWO52), STATUS_OK",
     "return sign | ((e + 1076) << 52) | (m - _TWO52), STATUS_OK", "f64"),             # exponent bias
    ("oracle/exact.py", "e = max(floor_log2_ratio(N, D) - 52, -1074)",
     "e = max(floor_log2_ratio(N, D) - 52, -1073)", "f64"),                            # subnormal limit
    ("oracle/exact.py", "e = max(floor_log2_ratio(N, D) - 52, -1074)",
     "e = max(floor_log2_ratio(N, D) - 53, -1074)", "f64"),                            # precision
    ("oracle/exact.py", "    if twice > den or (twice == den and (m & 1)):\n        m += 1\n    # Step 7",
     "    if twice >= den:\n        m += 1\n    # Step 7", "f64"),                      # ties away from zero
    ("oracle/exact.py", "    if twice > den or (twice == den and (m & 1)):\n        m += 1\n    # Step 7",
     "    if twice > den:\n        m += 1\n    # Step 7", "f64"),                       # ties down
    ("oracle/exact.py", "    if m == _TWO53:\n        m = _TWO52\n        e += 1\n    if m >= _TWO52 and e + 52 > 1023",
     "    if m >= _TWO52 and e + 52 > 1023", "f64"),                                    # binade carry
    ("oracle/exact.py", "if m >= _TWO52 and e + 52 > 1023:", "if m >= _TWO52 and e + 52 > 1024:", "f64"),  # overflow
    ("oracle/exact.py", "if Q + k - 1 >= 309:", "if Q + k - 1 >= 308:", "f64"),        # range cut (inf)
    # range cut (zero); "<= -324" would be an equivalent mutant (10^-324 < 2^-1075 too)
    ("oracle/exact.py", "if Q + k <= -325:", "if Q + k <= -323:", "f64"),
    ("oracle/exact.py", "    return t if ge else t - 1", "    return t", "all"),         # floor log2
    ("oracle/exact.py", "Q = Q + (len(s) - len(t))", "Q = Q", "f64"),                  # trailing zeros
    ("oracle/exact.py", "        v = v * 10 ** len(part) + int(part)",
     "        v = v * 10 ** 4000 + int(part)", "all"),                                 # long significand chunks
    ("oracle/exact.py", "    if len(s) <= 4000:\n        return int(s)",
     "    if len(s) <= 4000:\n        return int(s)\n    return int(s[:4000])", "all"),  # >4000 digits dropped
    ("oracle/exact.py", "    if lg <= emin - prec - 1:", "    if lg <= emin - prec:", "all"),  # hex zero cut
    ("oracle/exact.py", "    if lg >= emax + 1:", "    if lg >= emax:", "all"),        # hex inf cut
    ("oracle/lexer.py", "        exp = int_of_digits(\"\".join(exp_digits))",
     "        exp = int_of_digits(\"\".join(exp_digits)[-4:])", "all"),                # exponent truncated
    ("oracle/lexer.py", "        if eneg:\n            exp = -exp", "        if eneg:\n            exp = exp", "all"),
    ("oracle/lexer.py", "    return (\"num\", neg, digits, exp - len(frac_digits))",
     "    return (\"num\", neg, digits, exp - len(int_digits))", "all"),              # Q = exp - fraction digits
]


def main():
    src = {f: open(f).read() for f in set(m[0] for m in MUTS)}
    survived = 0
    try:
        for f, a, b, region in MUTS:
            s = src[f]
            assert s.count(a) >= 1, (f, a)
            if region == "f64":
                head, tail = s.split("def round_decimal32", 1)
                assert head.count(a) >= 1, a
                new = head.replace(a, b, 1) + "def round_decimal32" + tail
            else:
                new = s.replace(a, b, 1)
            open(f, "w").write(new)
            r = subprocess.run([sys.executable, "-m", "pytest", *PINS, "-q", "-x", "-p", "no:randomly"],
                               capture_output=True, text=True)
            ok = r.returncode != 0
            survived += not ok
            print("FAILS   " if ok else "SURVIVES", "|", f, "|", b.strip().splitlines()[-1][:70], flush=True)
            open(f, "w").write(src[f])
    finally:
        for f, s in src.items():
            open(f, "w").write(s)
    print("%d of %d mutations survived" % (survived, len(MUTS)))
    sys.exit(1 if survived else 0)


if __name__ == "__main__":
    main()
