"""Probe: exact pass (tensor-core vs dp4a) time on a config, and agreement of the two."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, paper_1902_09465_b200 as ak
cfg = synth.config(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
n = min(cfg.n, int(sys.argv[2])) if len(sys.argv) > 2 else cfg.n
X = synth.points(cfg, 0, n); Q = synth.queries(cfg)
ix = ak.Index(torch.from_numpy(X).cuda())
Qd = torch.from_numpy(Q).cuda()
s = torch.cuda.current_stream()
for it in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); idx, dist = ix.exact_device(Qd, cfg.k); e1.record(); torch.cuda.synchronize()
print(cfg.name, "n", n, "q", cfg.q, "exact ms", e0.elapsed_time(e1), "mode", os.environ.get("AKNN_EXACT_DP4A", "mma"))
np.save(f"/tmp/exact_{os.environ.get('AKNN_EXACT_DP4A', 'mma')}.npy", np.stack([idx.cpu().numpy(), dist.cpu().numpy()]))
