import ctypes as C, sys, os, time, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_20693_b200 import _capi
L = _capi.load()
t = torch.empty(1 << 20).pin_memory()
print("torch pinned ->", L.sct_debug_pointer_type(C.c_void_p(t.data_ptr())))
p = C.c_void_p()
L.sct_host_alloc(C.byref(p), 1 << 22)
print("engine pinned ->", L.sct_debug_pointer_type(p))
d = torch.empty(1 << 20, device="cuda")
print("torch device ->", L.sct_debug_pointer_type(C.c_void_p(d.data_ptr())))
