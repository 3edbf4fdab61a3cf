import sys, time, numpy as np
sys.path.insert(0,'.')
import paper_2505_09727_b200 as E
from paper_2505_09727_b200 import systems as S
print(E.device_count())
for name in ['cfg1','cfg2','cfg3','cfg4']:
    c = S.config(name); pos,q,box = c.system()
    p = E.build_plan(box,'pswf',c.eps,c.r_c)
    s = E.ParticleSystem(box,q,pos)
    ef = E.evaluate(p,s, timings=True)
    ef = E.evaluate(p,s, timings=True)
    print(name, ef.energy, {k: round(v*1e3,3) for k,v in ef.timings.items()}, flush=True)
    t=time.time(); 
    for _ in range(3): ef2 = E.evaluate(p,s)
    print('  overlapped host-API', (time.time()-t)/3*1e3, 'ms', ef2.energy, flush=True)
