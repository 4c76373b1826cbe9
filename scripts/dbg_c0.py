import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
import paper_1711_03888_b200 as nbz
from paper_1711_03888_b200 import datagen
os.environ["NBZG_DECODE"] = "warp"
for spec, mode in [("C1", "sz-lv"), ("C1", "sz-lv-prx"), ("C0", "sz-lv-prx")]:
    fields = datagen.generate(spec)
    snap = nbz.ParticleSnapshot(*fields)
    res = nbz.compress(snap, mode, nbz.ErrorBoundSpec.relative(1e-4))
    torch.cuda.synchronize()
    print(spec, mode, "compressed", nbz.ratio(res.archive), flush=True)
    rec = nbz.decompress(res.archive, device=True)
    torch.cuda.synchronize()
    print("ok", flush=True)
