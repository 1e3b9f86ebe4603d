"""GPU: sage2_prepare's internal fork / join (the Q quantizer on a library side stream, joined before
Delta S; DESIGN.md section 9 "Short-N preprocessing") under concurrency and CUDA-graph capture.

* two prepare + attention pipelines on two user streams at once (they share the library's side
  stream) give bitwise the results of running them one after the other;
* a whole forward (prepare + attention) captured into a CUDA graph and replayed on fresh inputs gives
  bitwise the eager result (the fork / join events are captured as graph edges).
"""
import pytest
import torch

from paper_2411_10958_b200 import sage2, synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    sage2.lib()


def _forward(q, k, v, ws, out, causal=False):
    B, Hq, N, d = q.shape
    Hkv = k.shape[1]
    sage2.prepare(q, k, v, ws, causal=causal)
    sage2.attention(out, ws, B, Hq, Hkv, N, d, causal=causal)


@pytest.mark.parametrize("N,d,causal", [(1024, 128, False), (3000, 128, True), (1500, 64, False)])
def test_two_streams_concurrent_equal_sequential(N, d, causal):
    B, Hq, Hkv = 2, 8, 4
    ins = [synth.make_qkv(B, Hq, Hkv, N, d, kind="iid", seed=s, device="cuda") for s in (1, 2)]
    wss = [sage2.alloc_workspace(B, Hq, Hkv, N, d, causal=causal) for _ in range(2)]
    ref = [torch.empty_like(x[0]) for x in ins]
    for (q, k, v), ws, o in zip(ins, wss, ref):
        _forward(q, k, v, ws, o, causal)
    torch.cuda.synchronize()
    outs = [torch.full_like(x[0], float("nan")) for x in ins]
    streams = [torch.cuda.Stream() for _ in range(2)]
    for _ in range(3):                                  # several rounds: the side stream is reused
        for (q, k, v), ws, o, st in zip(ins, wss, outs, streams):
            st.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(st):
                _forward(q, k, v, ws, o, causal)
        for st in streams:
            torch.cuda.current_stream().wait_stream(st)
    torch.cuda.synchronize()
    for r, o in zip(ref, outs):
        assert torch.equal(r, o)


def test_cuda_graph_capture_of_forward():
    B, Hq, Hkv, N, d = 1, 8, 8, 2048, 128
    q, k, v = synth.make_qkv(B, Hq, Hkv, N, d, kind="structured", seed=3, device="cuda")
    ws = sage2.alloc_workspace(B, Hq, Hkv, N, d)
    eager = torch.empty_like(q)
    _forward(q, k, v, ws, eager)
    torch.cuda.synchronize()
    sq, sk, sv = torch.zeros_like(q), torch.zeros_like(k), torch.zeros_like(v)
    gout = torch.empty_like(q)
    g = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):                       # capture on a non-default stream
        _forward(sq, sk, sv, ws, gout)                  # warm-up outside the graph
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=side):
            _forward(sq, sk, sv, ws, gout)
    sq.copy_(q)
    sk.copy_(k)
    sv.copy_(v)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(gout, eager)
