import os, sys, time
sys.path.insert(0, os.getcwd())
import torch, workloads as W
from paper_2512_23183_b200 import lq
w = W.config3()
lq.lq_vqe_adam(w.n, w.gates, w.theta, w.terms, max_iter=1)
for rep in range(2):
    torch.cuda.synchronize(); t=time.perf_counter()
    th, tr, T = lq.lq_vqe_adam(w.n, w.gates, w.theta, w.terms, max_iter=200, tol=0.0)
    torch.cuda.synchronize(); print(os.environ.get("TAG",""), "ms/iter", (time.perf_counter()-t)*1e3/(T+1))
t=time.perf_counter()
for _ in range(50): lq.lq_param_shift_grad(w.n, w.gates, w.theta, w.terms)
print(os.environ.get("TAG",""), "psr ms", (time.perf_counter()-t)*1e3/50)
