"""One MapElites generation inside cudaProfilerStart/Stop (ncu --profile-from-start off).

usage: python tools/one_generation.py CONFIG BATCH [WARM_GENERATIONS=2]
The profiled generation is generation WARM + 1 of a fresh run (seed 1); the
bench times generations 6..25 by default, so profile with WARM >= 5.
"""
import sys
sys.path.insert(0, ".")
import torch
import paper_2605_10128_b200 as P
from bench import grid_text
cfg = sys.argv[1]; B = int(sys.argv[2]); warm = int(sys.argv[3]) if len(sys.argv) > 3 else 2
g = P.grid_from_json_text(grid_text(cfg)); ctx = P.DcContext(g, P.build_action_set(g))
sess = P.QdSession(ctx, P.QdConfig(batch_size=B, iters_per_epoch=1 << 30))
sess.step(warm); torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
sess.step(1); torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
