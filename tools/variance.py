# per-application wall time distribution of the filter (host buffers), with
# NVML SM-clock / power / event-reason samples inside each application
import sys, threading, time
import numpy as np
sys.path.insert(0, '.')
import pynvml as nv
import paper_1605_08771_b200 as P
n, p, nc, streams, reps = (int(a) for a in sys.argv[1:6])
ctx = P.default_context()
A = np.asfortranarray(np.random.default_rng(0).standard_normal((n, n))); A = 0.5 * (A + A.T) / np.sqrt(n)
X = np.asfortranarray(np.random.default_rng(1).standard_normal((n, p)))
f = P.FilterApplier(A, P.build_contour_rule(P.SearchInterval(-0.3, 0.2), nc), ctx=ctx)
ctx.set_streams(streams)
Y = np.zeros_like(X, order="F")
nv.nvmlInit(); h = nv.nvmlDeviceGetHandleByIndex(0)
samples = []; stop = threading.Event()
def run():
    while not stop.is_set():
        samples.append((time.perf_counter(), nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM),
                        nv.nvmlDeviceGetPowerUsage(h) / 1e3, nv.nvmlDeviceGetCurrentClocksEventReasons(h)))
        time.sleep(0.005)
th = threading.Thread(target=run, daemon=True); th.start()
for _ in range(3): f.apply(X, out=Y)
win = []
for _ in range(reps):
    t0 = time.perf_counter(); f.apply(X, out=Y); t1 = time.perf_counter(); win.append((t0, t1))
stop.set(); th.join()
S = np.array([(t, c, pw, r) for t, c, pw, r in samples])
for t0, t1 in win:
    m = (S[:, 0] >= t0) & (S[:, 0] < t1)
    s = S[m]
    rs = int(np.bitwise_or.reduce(s[:, 3].astype(np.int64))) if len(s) else 0
    print(f"{1e3*(t1-t0):6.1f} ms  clk min {s[:,1].min() if len(s) else 0:.0f} med {np.median(s[:,1]) if len(s) else 0:.0f}  "
          f"power max {s[:,2].max() if len(s) else 0:.0f} W  reasons 0x{rs:x}", flush=True)
