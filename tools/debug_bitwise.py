"""Debug helper: where do GPU and oracle CVD results differ bitwise (cfg1 it0)?"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import oracle as O
from inputs import configs
import paper_2309_13824_b200 as T

c = configs.load(1)
ctx = T.Context(0)
ctx.tm_set_domain(c.box, torch.from_numpy(c.phi).cuda(), None, None, c.n)
x, y = torch.from_numpy(c.x).cuda(), torch.from_numpy(c.y).cuda()
ctx.tm_grid_bin(x, y)
xh, yh = torch.empty_like(x), torch.empty_like(y)
ctx.tm_cvd_step(None, xh, yh)
ctx.tm_sync()
o = O.iteration(O.FieldSet.from_config(c), c.x, c.y, "cvd")
gx, gy = xh.cpu().numpy(), yh.cpu().numpy()
bad = np.nonzero((gx != o.x_hat) | (gy != o.y_hat))[0]
print("x_hat mismatches:", len(bad))
cl = O.cells(O.FieldSet.from_config(c), c.x, c.y)
for i in bad[:6]:
    la, lb, vx, vy = cl.cell(i)
    print(i, "gpu", gx[i] - c.x[i], gy[i] - c.y[i], "or", o.x_hat[i] - c.x[i], o.y_hat[i] - c.y[i])
    print("   oracle ring", list(zip(la.tolist(), lb.tolist())))
    # sequential shoelace in oracle order, and in reverse, to see which the GPU matches
    def cen(vx, vy):
        S2 = sx = sy = 0.0
        n = len(vx)
        for k in range(n):
            k1 = (k + 1) % n
            cr = vx[k] * vy[k1] - vx[k1] * vy[k]
            S2 += cr; sx += cr * (vx[k] + vx[k1]); sy += cr * (vy[k] + vy[k1])
        return sx / (3.0 * S2), sy / (3.0 * S2)
    for r in range(len(vx)):
        a = cen(np.roll(vx, -r), np.roll(vy, -r))
        if a[0] == gx[i] - c.x[i] or (c.x[i] + a[0]) == gx[i]:
            print("   gpu matches rotation", r)
