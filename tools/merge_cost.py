"""Device cost of the island archive merge for N islands on one GPU (the
allgathered blobs are simulated by N copies of this island's blob)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2605_10128_b200 as P  # noqa: E402
from tools.synth_grid import config_json  # noqa: E402

text = config_json("cfg2")
g = P.grid_from_json_text(text)
ctx = P.DcContext(g, P.build_action_set(g))
sess = P.QdSession(ctx, P.QdConfig(batch_size=4096, iters_per_epoch=1 << 30))
sess.step(20)
nb = sess.blob_bytes()
stream = torch.cuda.ExternalStream(P.context_stream(ctx))
for n in (1, 2, 4, 8):
    blobs = torch.empty(n * nb, dtype=torch.uint8, device="cuda")
    with torch.cuda.stream(stream):
        for i in range(n):
            sess.pack(blobs[i * nb:].data_ptr())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(3):
            sess.merge(blobs.data_ptr(), n)
        e0.record(stream)
        for _ in range(20):
            sess.pack(blobs.data_ptr())
            sess.merge(blobs.data_ptr(), n)
        e1.record(stream)
    torch.cuda.synchronize()
    print(f"islands={n} blob={nb / 1e6:.2f} MB pack+merge {e0.elapsed_time(e1) / 20 * 1000:.1f} us", flush=True)
