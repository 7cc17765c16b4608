import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O, synth as S
from paper_2409_18772_b200 import lrqmm as L
lib = L.load_library()
dev = "cuda:0"
cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
for (rows, K, W) in [(257, 4096, 40), (256, 4096, 40), (128, 4096, 40), (257, 256, 40), (257, 4096, 32), (128, 512, 64), (128,256,64), (128, 288, 64)]:
    X = S.gen_matrix("normal", rows, K, 0); codes, lam = O.quantize(X, 4); R = O.residual(X, codes, lam)
    P = np.random.default_rng(1).standard_normal((K, W)).astype(np.float32)
    out = torch.zeros((rows, W), device=dev)
    x, l, p = cu(X), cu(lam), cu(P)
    st = torch.cuda.current_stream().cuda_stream
    rc = lib.lrqmm_debug_proj(0, x.data_ptr(), K, rows, K, l.data_ptr(), 4, 0, p.data_ptr(), None, W, out.data_ptr(), None, st)
    o = out.cpu().numpy(); ref = R @ P
    e = np.abs(o-ref); rowerr = e.max(axis=1); colerr = e.max(axis=0)
    print((rows,K,W), "rc", rc, "rel", np.linalg.norm(o-ref)/np.linalg.norm(ref), "bad rows", np.nonzero(rowerr>1e-3)[0][:10], "bad cols", np.nonzero(colerr>1e-3)[0][:40])
