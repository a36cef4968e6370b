import sys, os, json
sys.path.insert(0, os.getcwd())
import paper_2009_10400_b200 as tg
from paper_2009_10400_b200 import configs
p = configs.cfg5_h8(252, steps=400)
for P, r in ((8, 0), (2, 0)):
    e = tg.Engine(p, nranks=P, rank=r); e.peer_attach_solo(); e.step(20)
    try: e.sync()
    except tg.TveError: pass
    pk = e.profile_kernels(30)
    print(P, r, {k: round(v*1e3, 1) for k, v in pk.items()}, flush=True)
    e.close()
q = configs.cfg5_h8(126, steps=400)
e = tg.Engine(q); e.step(20); print("single 126^3", {k: round(v*1e3, 1) for k, v in e.profile_kernels(30).items()})
