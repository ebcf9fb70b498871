import sys; sys.path.insert(0,'.')
from paper_1805_11775_b200 import _native
import paper_1805_11775_b200 as P
lib=_native.lib()
for prec in (32,64):
    pl=_native.get_plan(3,1024,1024,9,True,prec,'hann',1,0)
    print(prec, 'kind', lib.hos_plan_k2_kind(pl.handle), 'nctas', lib.hos_plan_nctas(pl.handle))
