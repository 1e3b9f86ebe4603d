import ctypes, torch
torch.cuda.init()
L = ctypes.CDLL("paper_2411_10958_b200/libsage2.so")
for d in (64,128):
    for c in (0,1):
        out = (ctypes.c_int*6)()
        rc = L.sage2_debug_kernel_attrs(d, c, out)
        print(d, c, rc, list(out))
