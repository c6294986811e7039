"""Generate the golden fixtures in tests/golden/ from the REFERENCE ITSELF.

Runs the reference's own exec::run (oracle/_ref/libstencilc_ref.so, compiled from
/root/reference/proj/src by oracle/Makefile) on small seeded problems and stores the
results.  Run here (where /root/reference exists):  python tests/golden/make_golden.py
The fixtures are committed; nothing on the GPU box reads /root/reference.
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import bindings as O  # noqa: E402

CASES = [
    # name, shape, so, steps, damp_max, damp_width, hetero velocity, random initial levels
    ("c1_64_so2", (64, 64, 64), 2, 100, 0.0, 10, False, False),  # BASELINE config 1 (full)
    ("small_so2_damp", (12, 13, 14), 2, 9, 0.05, 3, True, True),
    ("small_so4", (14, 15, 16), 4, 8, 0.0, 10, True, True),
    ("small_so8_damp", (18, 20, 22), 8, 12, 0.05, 4, True, True),
    ("small_so12", (20, 21, 22), 12, 6, 0.02, 3, True, True),
    ("small_so16_damp", (22, 24, 26), 16, 6, 0.05, 4, True, True),
]


def receivers_for(shape, so):
    h = so // 2
    x, y = shape[0] // 2, shape[1] // 2 + shape[1] // 8
    return np.array([[x, y, z] for z in range(h, shape[2] - h)], np.int32)


def main():
    meta = {}
    for name, shape, so, steps, dmax, dw, hetero, rnd in CASES:
        rng = np.random.default_rng(1234)
        vel = (1500.0 + 1500.0 * rng.random(shape)).astype(np.float32) if hetero else None
        init = [(1e-3 * rng.standard_normal(shape)).astype(np.float32) for _ in range(3)] if rnd else None
        cfg = O.OracleConfig(shape=shape, space_order=so, steps=steps, velocity_field=vel,
                             damp_max=dmax, damp_width=dw)
        rec = receivers_for(shape, so)
        out = O.ref_run(cfg, initial_u=init, receivers=rec)
        info = O.ref_info(cfg)
        levels = out["levels"]
        rec_arr = dict(step_max_abs=out["step_max_abs"], rec_traces=out["rec_traces"], receivers=rec,
                       wavelet=info["wavelet"], dt=np.float32(info["dt"]))
        if vel is not None:
            rec_arr["velocity"] = vel
        if init is not None:
            rec_arr["initial_u"] = np.stack(init)
        if levels.size <= 3 * 20000:
            rec_arr["levels"] = levels
        np.savez_compressed(os.path.join(HERE, name + ".npz"), **rec_arr)
        meta[name] = dict(shape=shape, space_order=so, steps=steps, damp_max=dmax, damp_width=dw,
                          hetero=hetero, random_init=rnd, point_updates=out["point_updates"],
                          final_level=out["final_level"],
                          levels_sha256=[hashlib.sha256(levels[l].tobytes()).hexdigest() for l in range(3)],
                          source_point=list(info["source_point"]),
                          weights=[list(w) for w in info["weights"]],
                          flops_basic=info["flops_basic"], flops_aggressive=info["flops_aggressive"],
                          iet_hash_basic=str(info["iet_hash_basic"]),
                          iet_hash_aggressive=str(info["iet_hash_aggressive"]))
        print(name, out["point_updates"], out["wall_seconds"])
    # Known-answer values from SPEC.md (reproduced by the reference build).
    kat = {}
    for so in (2, 4, 8, 12, 16):
        i = O.ref_info(O.OracleConfig(shape=(256, 256, 256) if so == 8 else (32, 32, 32),
                                      space_order=so, steps=3))
        kat[str(so)] = dict(dt=float(np.float32(i["dt"])), weights=[list(w) for w in i["weights"]],
                            flops_basic=i["flops_basic"], flops_aggressive=i["flops_aggressive"],
                            source_point=list(i["source_point"]))
    meta["kat"] = kat
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(meta, f, indent=1)


if __name__ == "__main__":
    main()
