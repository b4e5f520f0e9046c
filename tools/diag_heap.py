"""Diagnose: spmm on torch tensors vs on fabric-heap memory (cfg3)."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2311_18141_b200 as rd  # noqa: E402
from paper_2311_18141_b200 import _lib as L  # noqa: E402


def timeit(fn, it=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it


a = rd.rmat(22, 16, seed=1)
b = rd.random_dense(a.cols, 128, 2)
c = torch.zeros((a.rows, 128), device="cuda")
print("torch tensors, czero:", timeit(lambda: rd.spmm_local(a, b, c, c_zero=True)))
print("torch tensors, acc  :", timeit(lambda: rd.spmm_local(a, b, c, c_zero=False)))
dev = (C.c_int * 1)(0)
cfg = L.FabricConfig(1, 6, 6 << 30, 4096, 0, 0, 1, dev, None)
f = C.c_void_p()
L.check(L.rdmm_fabric_create(C.byref(cfg), C.byref(f)), "create")
ptrs = []
for nbytes in (b.numel() * 4, c.numel() * 4):
    g = L.Gptr()
    L.check(L.rdmm_heap_alloc(f, 0, nbytes, C.byref(g)), "alloc")
    p = C.c_void_p()
    L.check(L.rdmm_gptr_device(f, 0, g, C.byref(p)), "dev")
    ptrs.append(p.value)
L.check(L.rdmm_memcpy(ptrs[0], b.data_ptr(), b.numel() * 4, None), "cp")
fl = C.c_uint64()
s = torch.cuda.current_stream().cuda_stream


def heap_call(cz):
    L.check(L.rdmm_spmm_csr_ex(4, a.rows, a.cols, 128, a.nnz, a.row_ptr.data_ptr(),
                               a.col_idx.data_ptr(), a.values.data_ptr(), ptrs[0], 128, ptrs[1],
                               128, 1 if cz else 0, None, 0, s, C.byref(fl)), "spmm")


print("heap B/C, czero     :", timeit(lambda: heap_call(True)))
print("heap B/C, acc       :", timeit(lambda: heap_call(False)))
import threading  # noqa: E402

res = []
th = threading.Thread(target=lambda: res.append(timeit(lambda: heap_call(True))))
th.start()
th.join()
print("heap B/C, czero, new thread:", res)
L.rdmm_fabric_destroy(f)
