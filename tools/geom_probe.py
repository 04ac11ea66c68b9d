import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2603_07156_b200 import _lib
import ctypes as C
for n in (4096, 10000, 16384, 50000):
    ctx = C.c_void_p()
    ld = ((n + 31) // 32) * 32
    st = _lib.lib.otb_create(C.byref(ctx), n, n, 0, n, ld, 0, None)
    print(n, st, _lib.lib.otb_last_error().decode() if st else "ok", flush=True)
    if st == 0:
        o = (C.c_int64 * 24)()
        _lib.lib.otb_info(ctx, o)
        print("  nt ns cl colw nstage ncl grid:", list(o)[:7], flush=True)
        _lib.lib.otb_destroy(ctx)
