import sys, os, ctypes, torch
sys.path.insert(0, os.getcwd())
import paper_2411_01288_b200 as H
from paper_2411_01288_b200 import _lib
from paper_2411_01288_b200.runner import LayerRunner
L = _lib.lib()
E,k,D,Hd,N = 32,2,384,1536,16384
dev = torch.device("cuda")
p, x = H.make_random_params(E, D, Hd, D, "gelu", seed=1, n_tokens=N, dtype=torch.bfloat16, device=dev)
a = H.synthesize_routing(N, E, k, "uniform", 1).to_device(dev)
run = LayerRunner(p, N, k, dev, torch.bfloat16)
for _ in range(5):
    run.forward(x, a)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 8)()
L.hxm_debug_prologue_ts(buf)
t = list(buf)
print("phase ns:", [t[i+1]-t[i] for i in range(7)], "total", t[7]-t[0])
print("phase us:", [round((t[i+1]-t[i])/1000, 2) if 0 <= t[i+1]-t[i] < 10**9 else None for i in range(7)])
