"""Host enqueue time per pipelined HostTrainStep call (C3, 12 and 3 chunks) against the device
time per step: the host must stay ahead of the copies for the e2e step to reach its floor.

    python profiles/e2e_hostprobe.py
"""
import sys, time, torch
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
from paper_2509_24006_b200 import HostTrainStep, SlaConfig
H,N,d=12,32768,128
cfg=SlaConfig(k_h=5,k_l=10,phi="softmax")
shape=(1,H,N,d)
hs=[torch.randn(shape).bfloat16().pin_memory() for _ in range(4)]
hw=(torch.randn(H,d,d)*0.1).bfloat16().pin_memory()
ho=[torch.empty(shape,dtype=torch.bfloat16).pin_memory() for _ in range(4)]
hdw=torch.empty((H,d,d),dtype=torch.float32).pin_memory()
for chunks in (12, 3):
    hts=HostTrainStep(1,H,N,d,64,64,cfg,torch.bfloat16,"cuda",chunks=chunks,pipelined=True)
    f=lambda: hts(hs[0],hs[1],hs[2],hw,hs[3],ho[0],ho[1],ho[2],ho[3],hdw)
    for _ in range(3): f()
    hts.finish(); torch.cuda.synchronize()
    t=[]
    e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        a=time.perf_counter(); f(); t.append((time.perf_counter()-a)*1e3)
    hts.finish(); e1.record(); torch.cuda.synchronize()
    print(f"chunks {chunks}: host ms per call {[round(x,2) for x in t]}; device {e0.elapsed_time(e1)/10:.2f} ms/step", flush=True)
