# Mutation check for the binary32 oracle pins (run by hand: python tests/mutate_oracle_f32.py): each
# listed change to oracle/exact.py round_decimal32 must make tests/test_oracle_f32_pins.py fail.
import subprocess, sys, shutil
src = open('oracle/exact.py').read()
muts = [("return sign | ((e + 150) << 23) | (m - _TWO23), STATUS_OK", "return sign | ((e + 151) << 23) | (m - _TWO23), STATUS_OK"),
        ("e = max(floor_log2_ratio(N, D) - 23, -149)", "e = max(floor_log2_ratio(N, D) - 23, -148)"),
        ("    if twice > den or (twice == den and (m & 1)):\n        m += 1\n    if m == _TWO24:", "    if twice >= den:\n        m += 1\n    if m == _TWO24:"),
        ("if m >= _TWO23 and e + 23 > 127:", "if m >= _TWO23 and e + 23 > 128:"),
        ("if Q + k <= -46:", "if Q + k <= -45:"),
        ("e = max(floor_log2_ratio(N, D) - 23, -149)", "e = max(floor_log2_ratio(N, D) - 24, -149)")]
try:
    for a, b in muts:
        assert src.count(a) >= 1, a
        # mutate only the binary32 part (after the marker)
        head, tail = src.split("def round_decimal32", 1)
        open('oracle/exact.py', 'w').write(head + "def round_decimal32" + tail.replace(a, b, 1))
        r = subprocess.run([sys.executable, "-m", "pytest", "tests/test_oracle_f32_pins.py", "-q", "-x"], capture_output=True, text=True)
        print("FAILS" if r.returncode else "SURVIVES", "|", b[:60])
finally:
    open('oracle/exact.py', 'w').write(src)
