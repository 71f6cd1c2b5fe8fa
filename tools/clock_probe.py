"""Probe: per-iteration device time vs NVML clocks/throttle reasons/processes (C4)."""
import os, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, pynvml
import synth, paper_1902_09465_b200 as ak
pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0)
samples = []; stop = threading.Event()
def poll():
    while not stop.is_set():
        try:
            samples.append((time.perf_counter(), pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                            pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_MEM),
                            pynvml.nvmlDeviceGetPowerUsage(h) / 1000, pynvml.nvmlDeviceGetCurrentClocksEventReasons(h),
                            len(pynvml.nvmlDeviceGetComputeRunningProcesses(h))))
        except Exception as e:
            samples.append((time.perf_counter(), -1, -1, -1, -1, repr(e)))
        stop.wait(0.02)
cfg = synth.config(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
X = synth.points(cfg); Q = synth.queries(cfg)
al = torch.from_numpy(ak.alpha_table(cfg.n, cfg.delta, cfg.d, "theory")).cuda()
ix = ak.Index(torch.from_numpy(X).cuda()); Qd = torch.from_numpy(Q).cuda(); s = torch.cuda.Stream()
ix.query_device(Qd, cfg.k, cfg.h, cfg.delta, 0, al, stream=s); torch.cuda.synchronize()
t = threading.Thread(target=poll, daemon=True); t.start()
for it in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); e0.record(s)
    ix.query_device(Qd, cfg.k, cfg.h, cfg.delta, 0, al, stream=s)
    e1.record(s); torch.cuda.synchronize(); t1 = time.perf_counter()
    win = [x for x in samples if t0 <= x[0] <= t1]
    sm = [x[1] for x in win]; pw = [x[3] for x in win]; rs = set(x[4] for x in win); pr = set(x[5] for x in win)
    print("it %d dev %.1f ms  sm %s-%s  power %.0f-%.0f W  reasons %s procs %s" % (it, e0.elapsed_time(e1), min(sm, default=0), max(sm, default=0), min(pw, default=0), max(pw, default=0), [hex(r) for r in rs], pr), flush=True)
stop.set()
