"""C ABI: the library builds, loads and exports every symbol include/*.h declares
(-m "not gpu": no compute call without a GPU)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    names = []
    for f in os.listdir(os.path.join(ROOT, "include")):
        if f.endswith(".h"):
            src = open(os.path.join(ROOT, "include", f)).read()
            src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
            names += re.findall(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\*?\s*([A-Za-z_][A-Za-z0-9_]*)\s*\(",
                                src, flags=re.M)
    return sorted(set(names))


@pytest.fixture(scope="module")
def lib():
    from paper_2101_11408_b200 import build, native
    build.build()
    return native.load()


def test_exports_every_declared_symbol(lib):
    names = declared_functions()
    assert "parse_f64_batch" in names and "parse_f64_split" in names
    for name in names:
        assert hasattr(lib, name), name


def test_host_only_calls(lib):
    from paper_2101_11408_b200 import native
    assert b"sm_100a" in lib.fpp_version()
    assert lib.fpp_workspace_bytes_split(0) >= 256
    assert lib.fpp_workspace_bytes_batch(1000, 10) >= 256
    # argument validation happens before any CUDA call
    assert lib.parse_f64_batch(None, 10, None, 1, None, None, None) == native.FPP_EARG
    assert lib.parse_f64_batch(None, 0, None, -1, None, None, None) == native.FPP_EARG
    assert lib.parse_f64_split(None, 5, 0, None, 0, None, None, None, None) == native.FPP_EARG
    assert lib.parse_f64_split(ctypes.c_void_p(16), 5, 7, None, 0, ctypes.c_void_p(16), None, None,
                               None) == native.FPP_EARG


def test_oracle_and_product_are_independent():
    # the oracle imports nothing from the product package and vice versa
    for root, _d, files in os.walk(os.path.join(ROOT, "oracle")):
        for f in files:
            if f.endswith(".py"):
                txt = open(os.path.join(root, f)).read()
                assert not re.search(r"^\s*(import|from)\s+paper_2101_11408_b200", txt, re.M), f
    for root, _d, files in os.walk(os.path.join(ROOT, "paper_2101_11408_b200")):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".c")):
                txt = open(os.path.join(root, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f


def _table_words():
    path = os.path.join(ROOT, "paper_2101_11408_b200", "csrc", "tables", "pow5_128.inc")
    words = [int(x, 16) for x in re.findall(r"0x([0-9a-f]{16})ull", open(path).read())]
    assert len(words) == 2 * 651
    return lambda q: (words[2 * (q + 342)], words[2 * (q + 342) + 1])


def _golden_rows(name):
    rows = []
    for line in open(os.path.join(ROOT, "tests", "golden", name)):
        if line.startswith("#") or not line.strip():
            continue
        rows.append(line.rstrip("\n").split("\t"))
    return rows


def test_generated_tables_match_paper():
    """T[q] (the generated .inc the kernels compile) against EVERY word PAPER.md
    prints: tab:pospower q = 0..55 (L462-501), tab:tabnearone q = -1..-27
    (L711-750), tab:awayfromone q = -28..-40 (L850-882) -- 96 rows, 164 words
    (tests/golden/pow5_table_words.tsv, each row with its line) -- and Example
    1's T[57].hi (L535)."""
    T = _table_words()
    rows = _golden_rows("pow5_table_words.tsv")
    assert len(rows) == 96
    nwords = 0
    for q, first, second, table, line in rows:
        q = int(q)
        hi, lo = T(q)
        assert hi == int(first, 16), (q, table, line)
        assert lo == (0 if second == "-" else int(second, 16)), (q, table, line)
        nwords += 1 if second == "-" else 2
    assert nwords == 164
    assert sorted(int(r[0]) for r in rows) == list(range(-40, 56))
    assert T(57)[0] == 11754943508222875079  # Example 1
    assert all(T(q)[0] >> 63 == 1 for q in range(-342, 309))  # normalised (L453-456)


def test_reciprocal_inverses_match_paper():
    """tab:insane: for q in [-17, -3] with an odd reciprocal,
    the printed inverse is the reciprocal word's inverse modulo 2^64, the
    printed product is the high word of (reciprocal word x inverse), with the
    printed number of trailing zeros -- and the reciprocal word is T[q].hi.
    (The paper's argument that the second multiplication cannot end in 64 + 9
    zero bits, L776-779.)"""
    T = _table_words()
    rows = _golden_rows("pow5_reciprocal_inverses.tsv")
    assert len(rows) == 11
    for q, first, inv, prod, zeros, line in rows:
        q, first, inv, prod, zeros = int(q), int(first, 16), int(inv, 16), int(prod, 16), int(zeros)
        assert T(q)[0] == first, (q, line)
        assert (first * inv) % (1 << 64) == 1, (q, line)
        assert (first * inv) >> 64 == prod, (q, line)
        assert (prod & -prod).bit_length() - 1 == zeros, (q, line)


def test_exponent_formula_closed_form():
    # q + floor(log2 5^q) == (217706 q) >> 16 on (-400, 350)
    for q in range(-399, 350):
        if q >= 0:
            exact = q + (5 ** q).bit_length() - 1
        else:
            exact = q - (5 ** -q - 1).bit_length()  # q - ceil(log2 5^-q)
        assert (217706 * q) >> 16 == exact, q
