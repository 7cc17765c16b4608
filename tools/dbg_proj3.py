import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O, synth as S
from paper_2409_18772_b200 import lrqmm as L
lib = L.load_library()
dev = "cuda:0"
cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
bad = 0; tot = 0
for rep in range(3):
  for (rows, K, W) in [(257, 4096, 40), (2048, 4096, 24), (128, 4096, 40), (257, 4096, 32), (1000, 2048, 64)]:
    X = S.gen_matrix("normal", rows, K, rep); codes, lam = O.quantize(X, 4); l64 = lam.astype(np.float64)[:, None]
    R = np.clip(np.rint((l64 * X - codes) * 32768), -32767, 32767) / 32768 / l64  # Q15 as stored
    P = np.random.default_rng(1).standard_normal((K, W)).astype(np.float32)
    ref = R @ P
    for mode in (0, 1):
        if mode == 1:
            P = np.random.default_rng(2).standard_normal((rows, W)).astype(np.float32); ref = R.T @ P
        out = torch.zeros(ref.shape, device=dev)
        x, l, p = cu(X), cu(lam), cu(P)
        st = torch.cuda.current_stream().cuda_stream
        lib.lrqmm_debug_proj(mode, x.data_ptr(), K, rows, K, 4, 0, p.data_ptr(), None, W, out.data_ptr(), None, st)
        o = out.cpu().numpy()
        e = np.linalg.norm(o-ref)/np.linalg.norm(ref)
        tot += 1; bad += e > 1e-5
print("bad", bad, "of", tot)
