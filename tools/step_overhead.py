import sys, time, json; sys.path.insert(0,'.')
import torch
from paper_2112_09728_b200 import synth
from paper_2112_09728_b200.layout import GBufferPlanes, VplPlanes, PassConfig
from paper_2112_09728_b200.session import GuidingSession
dev=torch.device('cuda:0')
for (w,h) in [(256,256),(1920,1080)]:
    fr=[(GBufferPlanes.from_ref(g,device=dev),VplPlanes.from_ref(v,device=dev)) for g,v in synth.sequence(w,h,16,seed=0,device=dev)]
    s=GuidingSession(w,h,PassConfig(seed=0,spp=1),device=dev)
    for i in range(20): s.step(*fr[i%16], i%16)
    torch.cuda.synchronize()
    n=200
    e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    t0=time.perf_counter(); e0.record()
    for i in range(n): s.step(*fr[i%16], i%16)
    e1.record(); torch.cuda.synchronize(); t1=time.perf_counter()
    print(json.dumps({"w":w,"h":h,"gpu_ms":e0.elapsed_time(e1)/n,"wall_ms":(t1-t0)*1e3/n}))
