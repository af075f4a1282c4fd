"""Board power and SM clock while config-3 cycles run back to back for a few
seconds (nvidia-smi sampled every ~50 ms), and the cycle time over time:
python scripts/power_probe.py [seconds]"""
import os
import subprocess
import sys
import threading
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1410_6609_b200 import mg  # noqa: E402
from paper_1410_6609_b200 import workloads as W  # noqa: E402

secs = float(sys.argv[1]) if len(sys.argv) > 1 else 3.0
samples = []
stop = threading.Event()


def sampler():
    q = "power.draw,clocks.sm,clocks.mem,temperature.gpu,clocks_throttle_reasons.active"
    while not stop.is_set():
        out = subprocess.run(["nvidia-smi", "--query-gpu=" + q, "--format=csv,noheader,nounits",
                              "-i", "0"], capture_output=True, text=True).stdout.strip()
        samples.append((time.time(), out))
        time.sleep(0.05)


w = W.cfg3(512, seed=0, with_rhs=False)
st = torch.cuda.Stream()
s = mg.Multigrid(w.shape, w.h, w.bc_type, w.bc_value, min_coarse=8, stream=st)
s.set_rhs(W.uniform_rhs(w.shape, 0))
for _ in range(5):
    s.vcycle()
time.sleep(1.0)
th = threading.Thread(target=sampler)
th.start()
time.sleep(0.3)
t0 = time.time()
times = []
while time.time() - t0 < secs:
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(st)
    s.vcycle()
    b.record(st)
    b.synchronize()
    times.append((time.time() - t0, a.elapsed_time(b)))
stop.set()
th.join()
for k in range(0, len(times), max(1, len(times) // 12)):
    print("t=%.2fs cycle %.3f ms" % times[k])
for t, o in samples[::max(1, len(samples) // 15)]:
    print("t=%.2fs %s" % (t - t0, o))
s.close()
