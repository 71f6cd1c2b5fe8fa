"""Probe: host-visible cost of one C2 query call, device API vs host API, timing on/off."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, paper_1902_09465_b200 as ak
cfg = synth.config(2)
X = synth.points(cfg); Q = synth.queries(cfg)
al = ak.alpha_table(cfg.n, cfg.delta, cfg.d, "theory")
ix = ak.Index(torch.from_numpy(X).cuda())
Qd = torch.from_numpy(Q).cuda(); ald = torch.from_numpy(al).cuda()
s = torch.cuda.Stream()
for mode in ("dev_t0", "dev_t1", "host_t0", "host_t1", "dev_t1_default_stream"):
    for it in range(4):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        if mode.startswith("dev"):
            st = None if mode.endswith("default_stream") else s
            ix.query_device(Qd, cfg.k, cfg.h, cfg.delta, 0, ald, timing=mode != "dev_t0", stream=st)
        else:
            ix.query(Q, cfg.k, cfg.h, cfg.delta, 0, al, counts=False, timing=mode == "host_t1")
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
        if it == 3:
            st_ = ix.stats()
            print(mode, f"wall {dt*1e3:.1f} ms  ms_total {st_['ms_total']:.1f}  adv {st_['ms_advance']:.1f} sel {st_['ms_select']:.1f} cmp {st_['ms_compact']:.1f} fil {st_['ms_filter']:.1f} rounds {st_['rounds']}", flush=True)
