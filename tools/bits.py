import sys; sys.path.insert(0,'.')
import sg_configs as S
from paper_2210_14313_b200 import api
for i in (2,3,5):
    p=S.baseline_config(i)
    print(p.name, [x.hex() for x in api.integrate(p.d,p.L,p.rule,p.kind,p.c,p.w,p.u)])
