import sys, os
sys.path.insert(0, os.getcwd())
import paper_2505_09727_b200 as E
from paper_2505_09727_b200 import systems as S
c = S.config(sys.argv[1]); pos, q, box = c.system()
plan = E.build_plan(box, "pswf", c.eps, c.r_c, device=0)
s = E.ParticleSystem(box, q, pos)
for _ in range(4): E.evaluate(plan, s)
