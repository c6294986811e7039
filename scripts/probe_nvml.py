"""How fast NVML answers while K1 streams: timestamps and call durations of the bench's clock
sampler calls around a 1000-step run (bench.py's Clocks saw one sample per 50 ms region)."""
import sys
import threading
import time

sys.path.insert(0, ".")
import pynvml as nv

import paper_1912_00695_b200 as P

nv.nvmlInit()
h = nv.nvmlDeviceGetHandleByIndex(0)
t0 = time.perf_counter()
for name, fn in [("clock", lambda: nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)),
                 ("reasons", lambda: nv.nvmlDeviceGetCurrentClocksEventReasons(h))]:
    a = time.perf_counter()
    for _ in range(20):
        fn()
    print(f"idle {name}: {(time.perf_counter() - a) / 20 * 1e3:.3f} ms/call")

prob = P.make_wave_problem(P.WaveProblemConfig(shape=(256,) * 3, spacing=(10., 10., 10.), space_order=8,
                                               steps=1100))
op = P.Operator(prob)
op.apply(10, 0)
log, running = [], True


def poll():
    while running:
        a = time.perf_counter()
        c = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        b = time.perf_counter()
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        e = time.perf_counter()
        log.append((a - t0, b - a, e - b, c, r))
        time.sleep(0.002)


th = threading.Thread(target=poll, daemon=True)
th.start()
time.sleep(0.02)
ra = time.perf_counter() - t0
op.apply_async(1000, 10)
op.collect(1000)
rb = time.perf_counter() - t0
time.sleep(0.02)
running = False
th.join()
inside = [x for x in log if ra <= x[0] <= rb]
print(f"region {ra:.4f}..{rb:.4f} s ({(rb - ra) * 1e3:.1f} ms): {len(log)} samples, {len(inside)} inside")
for x in log[:60]:
    print(f"  t {x[0]:.4f} clock {x[1] * 1e3:.3f} ms reasons {x[2] * 1e3:.3f} ms -> {x[3]} MHz 0x{x[4]:x}")
