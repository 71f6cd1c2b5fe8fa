"""Probe: per-step device time of the graph-launched loop vs the host loop (C2)."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth, paper_1902_09465_b200 as ak
cfg = synth.config(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
X = synth.points(cfg); Q = synth.queries(cfg)
al = torch.from_numpy(ak.alpha_table(cfg.n, cfg.delta, cfg.d, "theory")).cuda()
ix = ak.Index(torch.from_numpy(X).cuda())
Qd = torch.from_numpy(Q).cuda()
s = torch.cuda.Stream()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for mode in (False, True, False):
    ts, builds, walls = [], 0, []
    import time
    for it in range(8):
        flush.zero_(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        t0 = time.perf_counter()
        ix.query_device(Qd, cfg.k, cfg.h, cfg.delta, 0, al, timing=mode, stream=s)
        walls.append(1e3 * (time.perf_counter() - t0))
        e1.record(s); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
        if it >= 2: builds += ix.stats()["graph_builds"]
    st = ix.stats()
    print("timing" if mode else "graph ", "min %.1f med %.1f max %.1f" % (min(ts[2:]), statistics.median(ts[2:]), max(ts[2:])),
          "walls", ["%.0f" % w for w in walls], "builds", builds, "kernels %.1f" % sum(st[k] for k in ("ms_init", "ms_select", "ms_filter", "ms_compact", "ms_advance", "ms_output")), flush=True)
