timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "domain_constants or cfg1 or adaptive_full_size" > gpurun_out/r3d_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/r3d_tests.log
timeout 300 python -c "
import torch, time, paper_2309_13824_b200 as T
from inputs import configs
c = configs.load(3); dev = torch.device('cuda', 0)
to = lambda a: None if a is None else torch.from_numpy(a).to(dev)
ctx = T.Context(0)
for r in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    ctx.tm_set_domain(c.box, to(c.phi), to(c.mu), to(c.rho), c.n)
    torch.cuda.synchronize(); print('set_domain ms', (time.perf_counter() - t) * 1e3)
" > gpurun_out/r3d_setdomain.log 2>&1
