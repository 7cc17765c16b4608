import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_18772_b200 import lrqmm as L
lib = L.load_library()
W = int(sys.argv[1]) if len(sys.argv) > 1 else 24
op = int(sys.argv[2]) if len(sys.argv) > 2 else 2
rng = np.random.default_rng(6)
Y = torch.from_numpy((rng.standard_normal((16384, W)) * np.linspace(10, 1, W)).astype(np.float32)).cuda()
G = torch.zeros((W, W), dtype=torch.float64, device="cuda"); T = torch.zeros((W, W), device="cuda")
st = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    lib.lrqmm_debug_small(op, Y.data_ptr(), 16384, W, 16, G.data_ptr(), T.data_ptr(), st)
torch.cuda.synchronize(); print("ok")
