"""Workload for the steady-state ncu capture (profiles/ncu_steady_*.csv): one operator stepping
n^3 at the given SO; ncu profiles a run of consecutive stencil launches after warm-up with
--cache-control none, so every launch sees the L2 state its predecessor left (u[t+1] stores kept
in L2 with evict_last, write-backs of the previous step's dirty lines) -- the DRAM bytes per
launch of the kernel in its real regime.  Example (scripts/ncu_steady.sh):
  ncu --cache-control none --clock-control none -k regex:k_tma -s 30 -c 12 \
      --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      python scripts/ncu_steady.py 8 256 [damp]"""
import sys
sys.path.insert(0, '.')
import paper_1912_00695_b200 as P

so = int(sys.argv[1]) if len(sys.argv) > 1 else 8
n = int(sys.argv[2]) if len(sys.argv) > 2 else 256
damped = len(sys.argv) > 3 and sys.argv[3] == "damp"
dm = 3 * 1500.0 / (10 * 10.0) / 1500.0 ** 2 if damped else 0.0
prob = P.make_wave_problem(P.WaveProblemConfig(shape=(n, n, n), spacing=(10., 10., 10.), space_order=so, steps=60,
                                               damp_max=dm, damp_width=10))
op = P.Operator(prob)
op.apply(50, 0)
op.close()
