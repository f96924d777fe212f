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


def test_generated_tables_match_paper():
    """T[q] against the words PAPER.md prints (tables pospower, tabnearone,
    awayfromone; Example 1's T[57].hi) -- parsed from the generated .inc."""
    path = os.path.join(ROOT, "paper_2101_11408_b200", "csrc", "tables", "pow5_128.inc")
    words = [int(x, 16) for x in re.findall(r"0x([0-9a-f]{16})ull", open(path).read())]
    assert len(words) == 2 * 651

    def T(q):
        return words[2 * (q + 342)], words[2 * (q + 342) + 1]

    golden = {  # PAPER.md L462-501 (tab:pospower), L711-750 (tab:tabnearone), L858-882 (tab:awayfromone)
        0: (0x8000000000000000, 0), 1: (0xa000000000000000, 0), 27: (0xcecb8f27f4200f3a, 0),
        28: (0x813f3978f8940984, 0x4000000000000000), 55: (0xd0cf4b50cfe20765, 0xfff4b4e3f741cf6d),
        47: (0x8c213d9da502de45, 0x4526f422cc340000), -1: (0xcccccccccccccccc, 0xcccccccccccccccd),
        -17: (0xb877aa3236a4b449, 0x09befeb9fad487c3), -27: (0x9e74d1b791e07e48, 0x775ea264cf55347e),
        -28: (0xfd87b5f28300ca0d, 0x8bca9d6e188853fc), -29: (0xcad2f7f5359a3b3e, 0x096ee45813a04330),
        -34: (0x84ec3c97da624ab4, 0xbd5af13bef0b113e), -40: (0x8b61313bbabce2c6, 0x2323ac4b3b3da015),
    }
    for q, hl in golden.items():
        assert T(q) == hl, q
    assert T(57)[0] == 11754943508222875079  # Example 1
    assert all(T(q)[0] >> 63 == 1 for q in range(-342, 309))  # normalised (L453-456)


def test_exponent_formula_closed_form():
    # q + floor(log2 5^q) == (217706 q) >> 16 on (-400, 350)
    for q in range(-399, 350):
        if q >= 0:
            exact = q + (5 ** q).bit_length() - 1
        else:
            exact = q - (5 ** -q - 1).bit_length()  # q - ceil(log2 5^-q)
        assert (217706 * q) >> 16 == exact, q
