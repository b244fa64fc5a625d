import ctypes, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2511_14102_b200 import _lib
lib = _lib.lib()
L, E, K, kmax = 2, 6, 2, 8
for staging in (1, 0):
    h = ctypes.c_void_p()
    _lib.check(lib.mspq_cache_create(L, E, K, kmax, 40, 0, ctypes.byref(h)))
    caps = (ctypes.c_int * L)(*([3] * L))
    s = torch.cuda.current_stream().cuda_stream
    _lib.check(lib.mspq_cache_configure(h, 0, 0, caps, 3, 2, 0.25, 0.75, s))
    _lib.check(lib.mspq_cache_set_staging(h, staging))
    v = _lib.CacheView()
    _lib.check(lib.mspq_cache_view_get(h, ctypes.byref(v)))
    gbuf = torch.zeros(E, dtype=torch.int32, device="cuda")
    class H:
        pass
    def scal():
        torch.cuda.synchronize()
        hs = [v.host_stat[i] for i in range(13)]
        class A:
            __cuda_array_interface__ = {"shape": (13,), "typestr": "<i4", "data": (v.scal, False), "version": 3}
        d = torch.as_tensor(A(), device="cuda").cpu().tolist()
        return hs, d
    _lib.check(lib.mspq_cache_begin_cycle(h, 2, s)); print("staging", staging, "begin", scal())
    tg = torch.tensor([[[0, 1], [2, 3], [4, 5]], [[0, 1], [2, 3], [4, 5]]], dtype=torch.int32, device="cuda")
    for l in range(L):
        _lib.check(lib.mspq_cache_verify_layer(h, l, 3, tg[l].contiguous().data_ptr(), gbuf.data_ptr(), s))
        print("  verify", l, scal())
    lib.mspq_cache_destroy(h)
