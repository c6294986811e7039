"""Roofline model of the paper's §3 (Eqs. 2-4), the reference's specified-but-absent
`roofline` module (src/CMakeLists.txt:9 lists roofline.cpp, which is not
in the tree).  Used to put the B200 measurements and the paper's V100/Titan Z tables on
one chart.

  Eq. 3  OI = FP32 ops / (memory transactions x 32 B)
  Eq. 4  performance = FP32 ops per invocation x timesteps / total time
  Eq. 2  attainable = min(sp_peak, bandwidth x OI)
"""
from __future__ import annotations

import math
import re
from dataclasses import dataclass
from typing import Iterable, List, Optional, Sequence, Tuple

TRANSACTION_BYTES = 32  # "each read or write transaction ... 32 bytes size" (§3)


@dataclass(frozen=True)
class DeviceSpec:
    """Table 1 row."""
    name: str
    bandwidth: float   # GB/s (aggregate)
    sp_peak: float     # GFLOP/s
    dp_peak: float = 0.0
    memory: float = 0.0

    def __post_init__(self):
        if not (self.bandwidth > 0 and self.sp_peak > 0):
            raise ValueError("device bandwidth and sp_peak must be positive")

    @property
    def ridge(self) -> float:
        return self.sp_peak / self.bandwidth


# Paper Table 1 (Titan Z uses the aggregate 672 GB/s, SPEC.md DESIGN DECISIONS) and the
# B200 of this pool (MEASURED_PEAKS.json copy bandwidth; FP32 CUDA-core peak
# 148 SMs x 128 lanes x 2 x 1.965 GHz).
V100 = DeviceSpec("Tesla V100", 900.0, 14000.0, 7000.0, 16.0)
TITAN_Z = DeviceSpec("GTX Titan Z", 672.0, 4746.0, 1568.0, 12.0)
B200 = DeviceSpec("B200 (measured copy BW)", 6534.1, 74449.0, 37225.0, 180.0)


@dataclass(frozen=True)
class ProfileRecord:
    """Tables 2-3 row."""
    space_order: int
    dse: str
    fp32_count: float          # per kernel invocation (one time step)
    mem_transactions: float    # 32-byte transactions per invocation
    total_time: float          # seconds for `timesteps` steps
    timesteps: int
    runs: int = 1

    def __post_init__(self):
        if self.fp32_count < 0 or self.mem_transactions < 0:
            raise ValueError("counts must be non-negative")
        if self.timesteps < 1:
            raise ValueError("timesteps must be >= 1")


@dataclass(frozen=True)
class RooflinePoint:
    oi: float
    performance: float
    attainable: float
    pct_of_attainable: float
    bound: str
    label: Tuple[int, str]


def operational_intensity(fp_ops: float, mem_transactions: float) -> float:
    """Eq. 3."""
    if mem_transactions <= 0:
        raise ValueError("memory transactions must be positive")
    return fp_ops / (mem_transactions * TRANSACTION_BYTES)


def performance(rec: ProfileRecord) -> float:
    """Eq. 4 under the x-timesteps interpretation: GFLOP/s."""
    if not rec.total_time > 0:
        raise ValueError("total time must be positive")
    return rec.fp32_count * rec.timesteps / rec.total_time / 1e9


def attainable_peak(dev: DeviceSpec, oi: float) -> float:
    """Eq. 2."""
    if not oi > 0:
        raise ValueError("oi must be positive")
    return min(dev.sp_peak, dev.bandwidth * oi)


def classify(dev: DeviceSpec, oi: float) -> str:
    """memory iff oi < ridge; the ridge itself counts as compute."""
    return "memory" if oi < dev.ridge else "compute"


def point(dev: DeviceSpec, rec: ProfileRecord) -> RooflinePoint:
    oi = operational_intensity(rec.fp32_count, rec.mem_transactions)
    perf = performance(rec)
    att = attainable_peak(dev, oi)
    return RooflinePoint(oi, perf, att, perf / att, classify(dev, oi), (rec.space_order, rec.dse))


def _num(text: str) -> float:
    """Numbers with thousands separators or comma decimals ("135,73")."""
    t = text.strip()
    if re.fullmatch(r"-?\d{1,3}(\.\d{3})+(,\d+)?", t):  # 1.450.112.268 or 1.234,5
        t = t.replace(".", "").replace(",", ".")
    elif re.fullmatch(r"-?\d+,\d{1,2}", t):  # 135,73 (comma decimal)
        t = t.replace(",", ".")
    else:
        t = t.replace(",", "").replace("_", "")
    return float(t)


def ingest_profiles(text: str) -> List[ProfileRecord]:
    """Parse `space_order,dse,fp32_count,mem_transactions,total_time_s,timesteps,runs` rows
    (header optional).  Fields may quote thousands separators.  Errors name the line."""
    out: List[ProfileRecord] = []
    for lineno, line in enumerate(text.splitlines(), 1):
        line = line.strip()
        if not line or line.startswith("#") or line.startswith("space_order"):
            continue
        fields = [f.strip().strip('"') for f in re.split(r',(?=(?:[^"]*"[^"]*")*[^"]*$)', line)]
        if len(fields) != 7:
            raise ValueError(f"line {lineno}: expected 7 fields, got {len(fields)}")
        try:
            rec = ProfileRecord(int(fields[0]), fields[1], _num(fields[2]), _num(fields[3]), _num(fields[4]),
                                int(_num(fields[5])), int(_num(fields[6])))
        except ValueError as e:
            raise ValueError(f"line {lineno}: {e}") from None
        out.append(rec)
    return out


def emit_chart(points: Sequence[RooflinePoint], dev: DeviceSpec, title: Optional[str] = None) -> Tuple[str, str]:
    """Log-log roofline SVG (bandwidth roof, compute roof, ridge, labelled points) plus the
    numeric `.dat` table backing it.  Returns (svg, dat)."""
    if not points:
        raise ValueError("need at least one point")
    W, Hh, m = 640, 420, 60
    xs = [p.oi for p in points] + [dev.ridge]
    ys = [p.performance for p in points] + [dev.sp_peak]
    x0, x1 = 10 ** math.floor(math.log10(min(xs) / 2)), 10 ** math.ceil(math.log10(max(xs) * 2))
    y0, y1 = 10 ** math.floor(math.log10(min(ys) / 2)), 10 ** math.ceil(math.log10(max(ys) * 2))

    def X(v):
        return m + (W - 2 * m) * (math.log10(v) - math.log10(x0)) / (math.log10(x1) - math.log10(x0))

    def Y(v):
        return Hh - m - (Hh - 2 * m) * (math.log10(v) - math.log10(y0)) / (math.log10(y1) - math.log10(y0))

    svg = [f'<svg xmlns="http://www.w3.org/2000/svg" width="{W}" height="{Hh}">',
           f'<text x="{W / 2}" y="20" text-anchor="middle">{title or "Roofline: " + dev.name}</text>',
           f'<line x1="{m}" y1="{Hh - m}" x2="{W - m}" y2="{Hh - m}" stroke="black"/>',
           f'<line x1="{m}" y1="{m}" x2="{m}" y2="{Hh - m}" stroke="black"/>']
    bw_lo = max(x0, y0 / dev.bandwidth)
    svg.append(f'<line x1="{X(bw_lo):.1f}" y1="{Y(dev.bandwidth * bw_lo):.1f}" x2="{X(dev.ridge):.1f}" '
               f'y2="{Y(dev.sp_peak):.1f}" stroke="blue"/>')
    svg.append(f'<line x1="{X(dev.ridge):.1f}" y1="{Y(dev.sp_peak):.1f}" x2="{X(x1):.1f}" y2="{Y(dev.sp_peak):.1f}" '
               f'stroke="red"/>')
    dat = ["# oi perf_gflops attainable_gflops pct_of_attainable bound label"]
    for p in points:
        svg.append(f'<circle cx="{X(p.oi):.1f}" cy="{Y(p.performance):.1f}" r="4" fill="black"/>')
        svg.append(f'<text x="{X(p.oi) + 6:.1f}" y="{Y(p.performance) - 6:.1f}" font-size="10">'
                   f'SO {p.label[0]} {p.label[1]} {100 * p.pct_of_attainable:.1f}%</text>')
        dat.append(f"{p.oi:.4f} {p.performance:.2f} {p.attainable:.2f} {p.pct_of_attainable:.4f} {p.bound} "
                   f"so{p.label[0]}_{p.label[1]}")
    svg.append("</svg>")
    return "\n".join(svg), "\n".join(dat) + "\n"


# The paper's Tables 2-3: (device, dse, so, fp32/invocation,
# memory transactions/invocation, execution time s for 30,000 steps, printed OI, printed GFLOP/s)
PAPER_TABLES = [
    ("titanz", "basic", 8, 1450112268, 22722746, 553.92, 1.99, 78.54),
    ("titanz", "basic", 12, 2013392118, 28068109, 854.39, 2.24, 70.70),
    ("titanz", "basic", 16, 2375372938, 29871728, 907.72, 2.48, 78.51),
    ("titanz", "basic", 24, 2898342158, 33348001, 1150.01, 2.71, 75.61),
    ("titanz", "aggressive", 8, 641887345, 22637047, 135.73, 0.89, 141.88),
    ("titanz", "aggressive", 12, 760134906, 27737029, 179.15, 0.86, 127.29),
    ("titanz", "aggressive", 16, 842931505, 29704549, 180.55, 0.89, 140.06),
    ("titanz", "aggressive", 24, 929761776, 32926331, 219.76, 0.88, 126.92),
    ("v100", "basic", 8, 1450996129, 9245436, 553.92, 4.90, 693.77),
    ("v100", "basic", 12, 2013446796, 9112947, 854.39, 6.90, 740.48),
    ("v100", "basic", 16, 2375384531, 7722032, 907.72, 9.61, 816.86),
    ("v100", "basic", 24, 2898311328, 11862338, 1150.01, 7.64, 719.60),
    ("v100", "aggressive", 8, 641882304, 9256098, 15.31, 2.18, 1258.16),
    ("v100", "aggressive", 12, 760133342, 9289727, 20.37, 2.56, 1119.42),
    ("v100", "aggressive", 16, 842930745, 8026245, 20.21, 3.28, 1251.51),
    ("v100", "aggressive", 24, 929760267, 11670483, 18.48, 2.49, 1509.60),
]


def paper_records(device: str) -> List[ProfileRecord]:
    return [ProfileRecord(so, dse, fp, tx, t, 30000, 5) for dev, dse, so, fp, tx, t, _, _ in PAPER_TABLES
            if dev == device]


def b200_record(space_order: int, form: str, gpts: float, dram_bytes_per_point: float,
                flops_per_point: int, timesteps: int = 1000, n: int = 256) -> ProfileRecord:
    """A B200 measurement (bench GPts/s + ncu DRAM bytes) as a Table-2/3-style record."""
    pts = (n - space_order) ** 3
    return ProfileRecord(space_order, form, flops_per_point * pts, dram_bytes_per_point * pts / TRANSACTION_BYTES,
                         pts * timesteps / (gpts * 1e9), timesteps)
