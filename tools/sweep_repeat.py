"""Live sweep launch times (CUDA events, tg_sweep_timing) of MapElites
generations and of repeated evaluations of one fixed batch (debug: how much
of the sweep time depends on the state the previous kernels leave)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2605_10128_b200 as P
from tools.synth_grid import config_json
cfg = sys.argv[1]; B = int(sys.argv[2])
g = P.grid_from_json_text(config_json(cfg)); ctx = P.DcContext(g, P.build_action_set(g))
sess = P.QdSession(ctx, P.QdConfig(batch_size=B, iters_per_epoch=1 << 30))
sess.step(2); torch.cuda.synchronize()
P.sweep_timing(ctx, True)
for i in range(4):
    sess.step(1); torch.cuda.synchronize()
    ms, n = P.sweep_timing(ctx, True)
    print(f"generation {i}: sweep {ms:.3f} ms over {n} launches", flush=True)
G = sess.offspring()
for i in range(4):
    ctx.evaluate_arrays(G, 3, 2); torch.cuda.synchronize()
    ms, n = P.sweep_timing(ctx, True)
    print(f"fixed batch eval {i}: sweep {ms:.3f} ms over {n} launches", flush=True)
