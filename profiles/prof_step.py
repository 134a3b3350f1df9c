"""One C3 fwd+bwd step loop for ncu captures (profiles/collect.sh): B=1, H=12, N=32768, d=128."""
import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_24006_b200 import SLA, SlaConfig
B,H,n,d = 1,12,32768,128
op = SLA(B,H,n,d,64,64,SlaConfig(k_h=5,k_l=10,phi="softmax"),torch.bfloat16)
g = torch.Generator(device='cuda').manual_seed(0); shape=(B,H,n,d)
q,k,v,do = (torch.randn(shape,generator=g,device='cuda').bfloat16() for _ in range(4))
w = (torch.randn((H,d,d),generator=g,device='cuda')*0.1).bfloat16()
for _ in range(int(sys.argv[1]) if len(sys.argv)>1 else 2):
    st = op.forward(q,k,v,w); gr = op.backward(st,q,k,v,w,do)
torch.cuda.synchronize(); print("done")
