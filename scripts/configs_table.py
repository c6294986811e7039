"""Measure every BASELINE.json config that fits one B200 (development/report script; the
driver's headline is bench.py).  Writes gpurun_out/configs.json.

  1  64^3 SO 2, 100 steps, source + receiver line: GPU (factorised, plain f64) vs the
     reference's exec::run on the host (all threads) -- the config the CPU runs as-is
  2  256^3 SO 4/8/12/16, 1000 steps (K1)
  3  256^3 SO 8/16: plain (basic DSE) FP32 and FP64 vs factorised -- GPts/s, reference flop
     counts, GFLOP/s (DRAM bytes per point come from ncu, profiles/)
  4  512^3 SO 8 with a damping layer (damp_width 10, damp_max 2e-5... as chosen below), 1 GPU
  5  512^3 SO 16 per GPU (K1; the temporal-blocking K3 was retired), 1 GPU, and
     512^3 at the other space orders
"""
import json, sys, time
import numpy as np
sys.path.insert(0, '.')
import paper_1912_00695_b200 as P

FL_A = {2: 24, 4: 34, 8: 57, 12: 75, 16: 93}
FL_B = {2: 69, 4: 105, 8: 165, 12: 225, 16: 285}
out = {}


def gpts(shape, so, nt, form="factorised", tb=1, damp_max=0.0, damp_width=10, warm=5):
    prob = P.make_wave_problem(P.WaveProblemConfig(shape=shape, spacing=(10., 10., 10.), space_order=so,
                                                   steps=nt + warm + 2, damp_max=damp_max, damp_width=damp_width))
    op = P.Operator(prob, form=form, time_block=tb)
    op.apply(warm, 0)
    r = op.apply(nt, warm)
    pts = np.prod([s - so for s in shape])
    v = pts * nt / r.device_seconds / 1e9
    op.close()
    return round(float(v), 2)


# ---- config 1 ----
from oracle import bindings as O
shape, so, nt = (64, 64, 64), 2, 100
prob = P.make_wave_problem(P.WaveProblemConfig(shape=shape, spacing=(10., 10., 10.), space_order=so, steps=nt))
rec = np.array([[32, 40, z] for z in range(1, 63)], np.int32)
c1 = {}
for form in ("factorised", "plain_f64"):
    op = P.Operator(prob, form=form, receivers=rec)
    op.apply(nt, 0)
    op2 = P.Operator(prob, form=form, receivers=rec)
    r = op2.apply(nt, 0)
    c1[form] = round(62 ** 3 * nt / r.device_seconds / 1e9, 3)
cfg = O.OracleConfig(shape=shape, space_order=so, steps=nt)
if O.ref_available():
    rr = O.ref_run(cfg, threads=0)
    c1["cpu_reference"] = round(rr["point_updates"] / rr["wall_seconds"] / 1e9, 4)
    c1["cpu_threads"] = O.omp_threads("ref")
out["config1_64cube_so2_100steps_gpts"] = c1
# ---- config 2 ----
out["config2_256cube_1000steps_gpts"] = {f"so{s}": gpts((256,) * 3, s, 1000) for s in (4, 8, 12, 16)}
# ---- config 3 ----
c3 = {}
for s in (8, 16):
    f = gpts((256,) * 3, s, 300)
    p32 = gpts((256,) * 3, s, 30, form="plain_f32", warm=2)
    p64 = gpts((256,) * 3, s, 30, form="plain_f64", warm=2)
    c3[f"so{s}"] = {"factorised": {"gpts": f, "flops_pt": FL_A[s], "gflops": round(f * FL_A[s], 1)},
                    "plain_f32": {"gpts": p32, "flops_pt": FL_B[s], "gflops": round(p32 * FL_B[s], 1)},
                    "plain_f64": {"gpts": p64, "flops_pt": FL_B[s], "gflops": round(p64 * FL_B[s], 1)},
                    "factorised_over_plain_f32": round(f / p32, 2)}
out["config3_256cube_plain_vs_factorised"] = c3
# ---- config 4 ----
# damping: damp_max = 3 c / (width h) * m-scale is the SURVEY suggestion; damp multiplies du/dt
# in m u_tt + damp u_t = lap u, so a rate ~ 3c/(width*h) * m = 3*1500/(10*10)/1500^2 ~ 2e-5
dm = 3 * 1500.0 / (10 * 10.0) / 1500.0 ** 2
out["config4_512cube_so8_damped_1gpu_gpts"] = {"damp_width": 10, "damp_max": dm,
                                               "gpts": gpts((512,) * 3, 8, 200, damp_max=dm, damp_width=10),
                                               "undamped_gpts": gpts((512,) * 3, 8, 200)}
# ---- config 5 ----
out["config5_512cube_so16_1gpu_gpts"] = {"k1": gpts((512,) * 3, 16, 100)}
out["k1_512cube_gpts"] = {f"so{s}": gpts((512,) * 3, s, 100) for s in (4, 8, 12, 16)}
print(json.dumps(out, indent=1))
import os
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/configs.json", "w"), indent=1)
