"""Small-solver kernels in isolation (for ncu / event timing):
python tools/prof_small.py W OP [N] [REPS]   (OP: 1 chol, 2 eig (separate kernels); 3, 4 the fused kernel)."""
import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_18772_b200 import lrqmm as L
lib = L.load_library()
W = int(sys.argv[1]) if len(sys.argv) > 1 else 24
op = int(sys.argv[2]) if len(sys.argv) > 2 else 2
n = int(sys.argv[3]) if len(sys.argv) > 3 else 16384
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
rng = np.random.default_rng(6)
# residual-like sketch: decaying spectrum with a few near-degenerate values
sv = np.sort(np.abs(rng.standard_normal(W)) + np.linspace(3, 0.5, W))[::-1]
Y = torch.from_numpy((rng.standard_normal((n, W)) * sv).astype(np.float32)).cuda()
G = torch.zeros((W, W), dtype=torch.float64, device="cuda"); T = torch.zeros((W, W), device="cuda")
st = torch.cuda.current_stream().cuda_stream
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for i in range(reps):
    if i == reps - 1: ev[0].record()
    assert lib.lrqmm_debug_small(op, Y.data_ptr(), n, W, 16, G.data_ptr(), T.data_ptr(), st) == 0
    if i == reps - 1: ev[1].record()
torch.cuda.synchronize()
print(f"W={W} op={op} n={n}: last call {ev[0].elapsed_time(ev[1]) * 1e3:.1f} us (incl. malloc/free)")
