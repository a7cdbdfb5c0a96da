"""ctypes binding of librqa_b200.so (include/rqa_b200.h).

The library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_2402_16853_b200/csrc``).  There is no CPU fallback: if the
library or a CUDA device is missing, calls raise DeviceError.
"""

import ctypes
import os
import threading

from .errors import DeviceError, InvalidArgument, SeriesTooShort

__all__ = ["lib", "LIB_PATH", "call", "SYMBOLS", "TIMING_SLOTS"]

LIB_PATH = os.environ.get("RQA_LIB_PATH") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "librqa_b200.so")  # RQA_LIB_PATH: A/B testing
TIMING_SLOTS = 11

_c = ctypes
_i32, _i64, _dbl, _vp = _c.c_int32, _c.c_int64, _c.c_double, _c.c_void_p
_pd = _c.POINTER(_c.c_double)
_pi64 = _c.POINTER(_c.c_int64)
_pi32 = _c.POINTER(_c.c_int32)

# symbol -> (restype, argtypes), one entry per declaration in include/rqa_b200.h
SYMBOLS = {
    "rqa_version": (_c.c_int, []),
    "rqa_device_count": (_c.c_int, []),
    "rqa_launch_counter": (_i64, []),
    "rqa_threshold": (_c.c_int, [_i32, _i32, _dbl, _pd]),
    "rqa_band_rows": (_c.c_int, [_i32, _i32, _i32, _i64, _pi64, _pi32]),
    "rqa_plan_units": (_c.c_int, [_i64, _i64, _i64, _i32, _i32, _i32, _pi32, _i64, _pi64]),
    "rqa_run": (_c.c_int, [_pd, _i64, _i32, _i32, _i32, _dbl, _i64, _i32, _pi64, _pi64,
                           _pi64, _pi64, _pd, _c.c_char_p, _c.c_size_t]),
    "rqa_run_prec": (_c.c_int, [_pd, _i64, _i32, _i32, _i32, _dbl, _i64, _i32, _i32, _i32,
                                _pi64, _pi64, _pi64, _pi64, _pi64, _pd, _c.c_char_p,
                                _c.c_size_t]),
    "rqa_run_multi": (_c.c_int, [_pd, _i64, _i32, _i32, _i32, _dbl, _i64, _i32, _pi32, _i32,
                                 _i32, _pi64, _pi64, _pi64, _pi64, _pi64, _pd, _c.c_char_p,
                                 _c.c_size_t]),
    "rqa_run_device_prec": (_c.c_int, [_vp, _i64, _i32, _i32, _i32, _dbl, _i64, _i32, _i64,
                                       _i64, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                       _c.c_char_p, _c.c_size_t]),
    "rqa_run_device": (_c.c_int, [_vp, _i64, _i32, _i32, _i32, _dbl, _i64, _i64, _i64, _i32,
                                  _vp, _vp, _vp, _vp, _vp, _vp, _vp, _c.c_char_p, _c.c_size_t]),
    "rqa_stitch_device": (_c.c_int, [_vp, _vp, _vp, _vp, _pi64, _i32, _i64, _vp, _vp,
                                     _c.c_char_p, _c.c_size_t]),
    "rqa_block": (_c.c_int, [_pd, _i64, _i32, _i32, _i32, _dbl, _i64, _i64, _i64, _i64, _i64,
                             _i32, _i32, _c.POINTER(_c.c_uint8), _c.c_char_p, _c.c_size_t]),
    "rqa_tile_scan": (_c.c_int, [_c.POINTER(_c.c_uint8), _i64, _i64, _i64, _i32, _pi64, _pi64,
                                 _pi64, _pi64, _i32, _c.c_char_p, _c.c_size_t]),
    "rqa_read_column": (_c.c_int, [_c.c_char_p, _c.c_char, _i64, _i64, _i32, _i32,
                                   _c.POINTER(_pd), _pi64, _pi64, _pi64, _pi64, _c.c_char_p,
                                   _c.c_size_t]),
    "rqa_free": (None, [_vp]),
    "rqa_fp64_peak": (_c.c_int, [_i32, _pd, _pd, _c.c_char_p, _c.c_size_t]),
    "rqa_release": (_c.c_int, []),
}

_lib = None
_lock = threading.Lock()


def lib():
    """Load librqa_b200.so once; raise DeviceError if it is absent."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise DeviceError(
                        f"{LIB_PATH} is missing: build it with "
                        "`python -c 'import __graft_entry__ as g; g.build()'` "
                        "(there is no CPU fallback)")
                handle = ctypes.CDLL(LIB_PATH)
                for name, (res, args) in SYMBOLS.items():
                    fn = getattr(handle, name)
                    fn.restype = res
                    fn.argtypes = args
                _lib = handle
    return _lib


def call(name: str, *args) -> None:
    """Call a status-returning entry point; map codes to the error hierarchy."""
    err = ctypes.create_string_buffer(512)
    rc = getattr(lib(), name)(*args, err, ctypes.sizeof(err))
    if rc == 0:
        return
    msg = err.value.decode(errors="replace") or f"{name} failed with code {rc}"
    if rc == -1:
        raise InvalidArgument(msg)
    if rc == -2:
        raise SeriesTooShort(msg)
    raise DeviceError(msg)
