"""TEST INFRASTRUCTURE — drives one libperfslice.so through the reference's
public C ABI (proj/include/perfslice.h) and prints the report texts as JSON.
Run once with the stock reference library (oracle/_ref/libperfslice.so) and
once with the same sources built with the GPU underneath
(integration/_build/public_abi/libperfslice.so); tests/test_gpu_public_abi.py
compares the two.  Each library runs in its own process: both define the same
symbols."""
from __future__ import annotations

import ctypes as C
import json
import sys


def main(lib_path: str, db: str, calls: list) -> None:
    lib = C.CDLL(lib_path)
    lib.ps_last_error.restype = C.c_char_p
    lib.ps_database_open.argtypes = [C.c_char_p, C.POINTER(C.c_void_p)]
    lib.ps_session_open.argtypes = [C.c_void_p, C.c_void_p, C.c_uint, C.POINTER(C.c_void_p)]
    lib.ps_iterations.argtypes = [C.c_void_p, C.c_char_p, C.c_double, C.c_int, C.POINTER(C.c_void_p)]
    lib.ps_congestion.argtypes = [C.c_void_p, C.c_char_p, C.c_char_p, C.c_uint, C.c_double, C.c_int,
                                  C.POINTER(C.c_void_p)]
    lib.ps_imbalance.argtypes = [C.c_void_p, C.c_char_p, C.c_double, C.c_int, C.POINTER(C.c_void_p)]
    lib.ps_string_free.argtypes = [C.c_void_p]
    lib.ps_session_close.argtypes = [C.c_void_p]
    lib.ps_database_close.argtypes = [C.c_void_p]
    h, s = C.c_void_p(), C.c_void_p()
    assert lib.ps_database_open(db.encode(), C.byref(h)) == 0, lib.ps_last_error()
    assert lib.ps_session_open(h, None, 0, C.byref(s)) == 0, lib.ps_last_error()
    out = []
    for call in calls:
        name, args = call[0], call[1:]
        p = C.c_void_p()
        if name == "iterations":
            st = lib.ps_iterations(s, args[0].encode(), args[1], args[2], C.byref(p))
        elif name == "congestion":
            st = lib.ps_congestion(s, args[0].encode(), args[1].encode(), args[2], args[3], args[4], C.byref(p))
        elif name == "imbalance":
            st = lib.ps_imbalance(s, args[0].encode(), args[1], args[2], C.byref(p))
        else:
            raise ValueError(name)
        text = C.cast(p, C.c_char_p).value.decode() if st == 0 else lib.ps_last_error().decode()
        if st == 0:
            lib.ps_string_free(p)
        out.append({"call": call, "status": st, "text": text})
    lib.ps_session_close(s)
    lib.ps_database_close(h)
    # psg kernel launches (libpsg.so is a dependency of the GPU build only)
    try:
        f = lib.psg_kernel_launches
        f.restype = C.c_uint64
        launches = int(f())
    except AttributeError:
        launches = None
    print(json.dumps({"results": out, "psg_kernel_launches": launches}))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], json.loads(sys.argv[3]))
