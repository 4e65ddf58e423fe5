import os, sys
sys.path.insert(0, '.')
import numpy as np, torch, gen, bench
import paper_2308_07173_b200 as g
sc, mp, T, T0 = gen.config_c3()
md = torch.from_numpy(np.array(mp)).cuda(); sd = torch.from_numpy(np.array(sc)).cuda()
im = g.build_index(md, 0.5); _, _, cm = g.knn_cov_self(im, 20, 1e-3); g.attach_cov(im, cm)
isc = g.build_index(sd, 0.0); _, _, cs = g.knn_cov_self(isc, 20, 1e-3)
print("align", flush=True)
Tr, info = g.align(sd, cs, im, cm, T0)
torch.cuda.synchronize()
print(info.iterations)
