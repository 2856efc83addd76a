"""Device time of one MapElites generation and of one plain evaluation (debug)."""
import sys, time
import torch
sys.path.insert(0, ".")
import paper_2605_10128_b200 as P
from tools.synth_grid import config_json
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
g = P.grid_from_json_text(config_json(cfg)); ctx = P.DcContext(g, P.build_action_set(g))
sess = P.QdSession(ctx, P.QdConfig(batch_size=B, iters_per_epoch=1 << 30))
st = torch.cuda.ExternalStream(P.context_stream(ctx))
sess.step(3); torch.cuda.synchronize()
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st); sess.step(1); e1.record(st); torch.cuda.synchronize()
    print("generation ms", e0.elapsed_time(e1), flush=True)
G = sess.offspring()
for _ in range(2):
    t0 = time.perf_counter(); ctx.evaluate_arrays(G, 3, 2); print("evaluate wall ms", (time.perf_counter() - t0) * 1e3, flush=True)
