"""B200-native (sm_100a) execution backend for Fireiron matrix-multiplication
strategies. The product is the native library ``_lib/libfireiron_b200.so``
(C ABI: include/fireiron_b200.h, C++ API: include/fireiron/*.hpp); this
package is its Python host binding."""
from ._native import FiError, lib, LIB_PATH  # noqa: F401
from .api import Plan, validate, elaborate, print_script, generate, plan_summary, check_async, host_snap  # noqa: F401
from . import strategies  # noqa: F401

__version__ = "0.1.0"
