import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O, synth as S
from paper_2409_18772_b200 import lrqmm as L
lib = L.load_library()
rows, K, W = 128, 32, 32
X = S.gen_matrix("normal", rows, K, 0); codes, lam = O.quantize(X, 4); R = O.residual(X, codes, lam)
P = np.random.default_rng(1).standard_normal((K, W)).astype(np.float32)
dev = "cuda:0"
cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
out = torch.full((rows, W), 7.0, device=dev)
x, l, p = cu(X), cu(lam), cu(P)
st = torch.cuda.current_stream().cuda_stream
rc = lib.lrqmm_debug_proj(0, x.data_ptr(), K, rows, K, l.data_ptr(), 4, 0, p.data_ptr(), None, W, out.data_ptr(), None, st)
torch.cuda.synchronize()
o = out.cpu().numpy(); ref = R @ P
print("rc", rc, "uniq(first 10)", np.unique(o)[:10], "nonzero", np.count_nonzero(o))
print("out[0,:6]", o[0,:6]); print("ref[0,:6]", ref[0,:6])
print("err", np.linalg.norm(o-ref)/np.linalg.norm(ref))
