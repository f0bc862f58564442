import sys
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np
import test_gpu_cma as T
import workloads as W
from gpu_helpers import q24
pair = T.CmaPair(16, 10, T._params(2))
for g in range(100):
    x = pair.gpu.ask(); f = pair.gpu.eval(W.ROSENBROCK, x); pair.gpu.tell(f)
    xh, fh = x.cpu().numpy(), f.cpu().numpy()
    o = pair.orc[0]; xo = o.ask()
    for r in range(1, 2): pair.orc[r].ask(); pair.orc[r].tell(fh[r])
    o.tell(fh[0])
    gm = pair.gpu.get("mean")[0].cpu().numpy(); gs = float(pair.gpu.get("sigma")[0])
    gc = pair.gpu.get("cov")[0].cpu().numpy(); ga = pair.gpu.get("chol")[0].cpu().numpy()
    gps = pair.gpu.get("p_sigma")[0].cpu().numpy()
    if g % 5 == 0 or g > 85:
        print(g, "x %.2e" % q24(xh[0], xo), "m %.2e" % q24(gm, o.m), "sig %.2e" % (abs(gs - o.sigma) / o.sigma),
              "C %.2e" % q24(gc.ravel(), o.C.ravel()), "A %.2e" % q24(ga.ravel(), o.A.ravel()),
              "ps %.2e" % q24(gps, o.p_sigma), "sigma %.3e" % o.sigma, "cond %.2e" % np.linalg.cond(o.C), "f %.3e" % fh[0].min())
