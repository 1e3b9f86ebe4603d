import ctypes, sys, torch
sys.path.insert(0, "/root/repo")
from paper_2411_10958_b200 import sage2, synth
B, H = 4, 32
N, d = int(sys.argv[1]), int(sys.argv[2])
q, k, v = synth.make_qkv(B, H, H, N, d, device="cuda")
ws = sage2.alloc_workspace(B, H, H, N, d)
sage2.prepare(q, k, v, ws)
out = torch.empty_like(q)
L = sage2.lib()
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
for fl in [int(x) for x in sys.argv[3].split(",")]:
    rc = L.sage2_attention(out.data_ptr(), B, H, H, N, d, fl, ws.data_ptr(), ctypes.c_size_t(ws.numel()), st)
    assert rc == 0
torch.cuda.synchronize()
