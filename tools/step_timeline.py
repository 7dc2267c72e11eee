"""Device/host timeline of bench.py's step (diagnostics): the same two-stream
step as bench.run_step, with CUDA events recorded on each variant's stream after
every API call and the host time at which each call returned. L2 flushed before
each step as in bench.py. Prints per marker the device time since the step
start and the host time since the step start (means over steps)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2405_02256_b200 as eu  # noqa: E402

gray, binary, dirs = bench.workload(0)
imgs = [torch.from_numpy(x).cuda() for x in bench.step_batches(gray, binary)]
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
cur = torch.cuda.current_stream()
streams = [torch.cuda.Stream(), torch.cuda.Stream()]
N = int(os.environ.get("STEPS", "20"))
acc_dev, acc_host = {}, {}
for it in range(N + 3):
    flush.fill_(1.0)
    marks = []

    def mark(name, st):
        e = torch.cuda.Event(enable_timing=True)
        e.record(st)
        marks.append((name, e, time.perf_counter()))

    mark("start", cur)
    for st in streams:
        st.wait_stream(cur)
    for v, (img, st) in enumerate(zip(imgs, streams)):
        with torch.cuda.stream(st):
            cx = eu.build_complex(img, "vertex", stream=st)
            mark(f"build[{v}]", st)
            cr = eu.critical_points(cx, stream=st)
            mark(f"critical[{v}]", st)
            r = eu.transforms(cr, dirs, elem_bytes="auto", share_heights=True, ht=(bench.HT_KERNEL, 1.0, "f64"),
                              stream=st)
            mark(f"transforms[{v}]", st)
    for st in streams:
        cur.wait_stream(st)
    mark("end", cur)
    torch.cuda.synchronize()
    if it >= 3:
        e0, h0 = marks[0][1], marks[0][2]
        for name, e, h in marks:
            acc_dev[name] = acc_dev.get(name, 0.0) + e0.elapsed_time(e)
            acc_host[name] = acc_host.get(name, 0.0) + (h - h0) * 1e3
print(f"{'marker':16s} {'device_ms':>10s} {'host_returned_ms':>16s}")
for k in acc_dev:
    print(f"{k:16s} {acc_dev[k] / N:10.3f} {acc_host[k] / N:16.3f}")
