import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "oracle"))
import oracle as O, paper_2411_01288_b200 as H
bf = torch.bfloat16
def dev(a, dt=torch.float32): return torch.as_tensor(np.asarray(a, np.float64)).to("cuda", dt)
def host(t): return t.detach().double().cpu().numpy()
def rnd(a): return host(dev(a, bf))
rng = np.random.default_rng(0)
for (E, n, d1, d2, blk) in [(1, 128, 64, 64, 1), (2, 300, 128, 256, 8), (32, 4096, 384, 1536, 8), (8, 1000, 128, 192, 3)]:
    a = rng.integers(0, E, n).astype(np.int32)
    x = rnd(rng.standard_normal((n, d1))); w = rnd(0.5*rng.standard_normal((E, d1, d2))); b = rng.standard_normal((E, d2))
    x2 = rnd(rng.standard_normal((n, d2)))
    orx = O.build_reindex(a, E, blk); rx = H.build_reindex(a, E, blk)
    y = H.esmm(dev(x, bf), dev(w, bf), dev(b), rx); torch.cuda.synchronize()
    print("esmm", E, n, d1, d2, O.scaled_err(host(y), O.esmm(x, w, b, orx)), flush=True)
    yt = H.esmm(dev(x2, bf), dev(w, bf), None, rx, w_transposed=True); torch.cuda.synchronize()
    print("esmm_T", O.scaled_err(host(yt), O.esmm(x2, np.ascontiguousarray(w.transpose(0,2,1)), None, orx)), flush=True)
    t = H.estmm(dev(x, bf), dev(x2, bf), rx); torch.cuda.synchronize()
    print("estmm", O.scaled_err(host(t), O.estmm(x, x2, orx)), flush=True)
