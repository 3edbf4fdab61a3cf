# K1/K3/sort stage times vs spread-bin edge S and sort sub-bins per bin edge
# usage: bash tools/spread_sweep.sh "cfg3 cfg5" "8:4 8:8 6:6"
for w in $1; do for cfg in $2; do S=${cfg%%:*}; D=${cfg##*:}; ESP_SPREAD_S=$S ESP_SORT_SUB=$D timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import paper_2505_09727_b200 as E
from paper_2505_09727_b200 import systems as S
c=S.config('$w'); pos,q,box=c.system()
p=E.build_plan(box,'pswf',c.eps,c.r_c,device=0); s=E.ParticleSystem(box,q,pos)
ts=[E.evaluate(p,s,timings=True).timings for _ in range(5)]
m=lambda k: min(t[k] for t in ts[1:])*1e3
print('$w S=$S sub=$D spread %.3f interp %.3f bin %.3f'%(m('spread'),m('interpolate'),m('bin')), flush=True)
"; done; done
