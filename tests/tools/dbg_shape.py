import sys; sys.path.insert(0, '/root/repo')
import torch
from paper_2509_24006_b200 import SLA, SlaConfig
n, d = int(sys.argv[1]), int(sys.argv[2])
g = torch.Generator(device="cuda").manual_seed(1)
mk = lambda: torch.randn((1, 1, n, d), generator=g, device="cuda").to(torch.bfloat16)
q, k, v, do = mk(), mk(), mk(), mk()
w = (torch.randn((1, d, d), generator=g, device="cuda") * 0.1).to(torch.bfloat16)
op = SLA(1, 1, n, d, 64, 64, SlaConfig(k_h=10.0, k_l=20.0, phi=sys.argv[3]), torch.bfloat16)
st = op.forward(q, k, v, w); torch.cuda.synchronize(); print("fwd ok", flush=True)
g2 = op.backward(st, q, k, v, w, do); torch.cuda.synchronize(); print("bwd ok", flush=True)
