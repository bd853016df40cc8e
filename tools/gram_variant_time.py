"""Time the Gram (k_gram_ws + reduce) of the bench's sample set with the librp that RP_LIBRP names;
one JSON line with the median ms and a checksum of G (compare variants with the default build)."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_1911_02373_b200 as rp

tag = sys.argv[1] if len(sys.argv) > 1 else "default"
dev = torch.device("cuda:0")
inp = bench.workload_inputs()
X = torch.from_numpy(inp["X"]).to(dev)
V = (rp.eval_metrics(inp["truth"], X) * torch.from_numpy(inp["noise"]).to(dev)).contiguous()
c, e = rp.xform_from_box(*rp.minmax(X))
G = rp.gram(X, V, inp["num"], inp["den"], c, e)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
ms = []
for _ in range(7):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    rp.gram(X, V, inp["num"], inp["den"], c, e, out=G)
    b.record()
    torch.cuda.synchronize()
    ms.append(a.elapsed_time(b))
print(json.dumps({"variant": tag, "gram_ms": statistics.median(ms), "G_sum": float(G.abs().sum().item()),
                  "G00": float(G[0, 0, 0].item())}), flush=True)
