"""B200-native batched decimal -> binary64 parser (arXiv 2101.11408).

The product is the CUDA library libfpparse.so (C ABI in include/fpparse.h);
native.py is its thin Python binding.  See DESIGN.md.
"""
from . import native  # noqa: F401
from .native import (parse_f64_batch, parse_f64_split, Workspace, FppError,  # noqa: F401
                     ST_OK, ST_OVERFLOW, ST_UNDERFLOW, ST_INVALID, ST_EMPTY)

__all__ = ["native", "parse_f64_batch", "parse_f64_split", "Workspace", "FppError",
           "ST_OK", "ST_OVERFLOW", "ST_UNDERFLOW", "ST_INVALID", "ST_EMPTY"]
