"""The C-ABI calls are stream-ordered and allocation-free, so a training step can be captured into
a CUDA graph: the forward's and backward's side-stream fork / join (summaries, column lists, dW)
and the programmatic-dependent launches must be capturable, and a replay must reproduce the eager
results bit for bit."""
import pytest
import torch

from paper_2509_24006_b200 import SLA, SlaConfig

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,d,heads", [(2048, 128, 2), (1024, 64, 3)])
def test_step_captures_into_a_cuda_graph(n, d, heads):
    g = torch.Generator(device="cuda").manual_seed(5)
    q, k, v, do = (torch.randn((1, heads, n, d), generator=g, device="cuda").bfloat16() for _ in range(4))
    w = (torch.randn((heads, d, d), generator=g, device="cuda") * 0.1).bfloat16()
    op = SLA(1, heads, n, d, 64, 64, SlaConfig(k_h=10.0, k_l=20.0, phi="softmax"), torch.bfloat16)
    shape = (1, heads, n, d)
    outs = dict(o=torch.empty(shape, dtype=torch.bfloat16, device="cuda"),
                o_s=torch.empty(shape, dtype=torch.bfloat16, device="cuda"),
                o_l=torch.empty(shape, dtype=torch.bfloat16, device="cuda"),
                lse=torch.empty(shape[:-1], dtype=torch.float32, device="cuda"),
                dq=torch.empty(shape, dtype=torch.bfloat16, device="cuda"),
                dk=torch.empty(shape, dtype=torch.bfloat16, device="cuda"),
                dv=torch.empty(shape, dtype=torch.bfloat16, device="cuda"),
                dw=torch.empty((heads, d, d), dtype=torch.float32, device="cuda"))
    state = op.new_state()

    def step():
        st = op.forward(q, k, v, w, state=state, out=(outs["o"], outs["o_s"], outs["o_l"], outs["lse"]))
        op.backward(st, q, k, v, w, do, out=(outs["dq"], outs["dk"], outs["dv"], outs["dw"]))

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step()  # eager reference (also warms up)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    want = {nm: t.clone() for nm, t in outs.items()}
    for t in outs.values():
        t.zero_()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        step()
    graph.replay()
    graph.replay()
    torch.cuda.synchronize()
    for nm, t in outs.items():
        assert torch.equal(t, want[nm]), nm
