import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1911_02373_b200 as rp, synth, oracle
fc = synth.fitheavy(sigma=0.01)
V = np.stack([np.asarray(v, dtype=np.float64) for v in oracle.program_metrics(fc.truths[0], fc.X)]) * fc.noise
X = torch.from_numpy(fc.X).cuda()
c, e = rp.xform_from_box(*rp.minmax(X))
for i in range(3):
    G = rp.gram(X, torch.from_numpy(V[i:i+1]).cuda(), fc.num_exp, fc.den_exp, c, e)[0].cpu().numpy()
    Go = np.asarray(oracle.gram(fc.X, V[i], fc.num_exp, fc.den_exp, c, e, nthreads=16), dtype=np.float64)
    dg = np.sqrt(np.outer(np.diag(Go), np.diag(Go)))
    print(i, np.max(np.abs(G - Go) / dg))
