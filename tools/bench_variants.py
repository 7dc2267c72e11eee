"""Which part of bench.py's timed loop inflates the step time? (diagnostics)"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench, paper_2405_02256_b200 as eu
gray, binary, dirs = bench.workload(0)
imgs = [torch.from_numpy(gray).cuda(), torch.from_numpy(binary).cuda()]
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
s = torch.cuda.current_stream()
for prof in (0, 1):
    for hold in (0, 1):
        res = None
        ts = []
        for it in range(13):
            flush.fill_(1.0)
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            if prof:
                eu.profile_enable(True)
            ev0.record(s)
            r = bench.run_step(eu, torch, imgs, dirs)
            if hold:
                res = r
            else:
                del r
            ev1.record(s)
            ev1.synchronize()
            if prof:
                eu.profile_read("k2_transforms")
                eu.profile_enable(False)
            if it >= 3:
                ts.append(ev0.elapsed_time(ev1))
        res = None
        print(f"prof={prof} hold={hold} step_ms={np.mean(ts):.3f} min={np.min(ts):.3f}")
