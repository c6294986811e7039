"""The roofline/report module against the SPEC examples and every cell of
the paper's Tables 2-3."""
import math

import pytest

from paper_1912_00695_b200 import roofline as R


def test_operational_intensity_examples():
    assert abs(R.operational_intensity(1450112268, 22722746) - 1.99) <= 0.01
    assert R.operational_intensity(32, 1) == 1.0
    assert abs(R.operational_intensity(1450996129, 9245436) - 4.90) <= 0.01
    with pytest.raises(ValueError):
        R.operational_intensity(1, 0)


@pytest.mark.parametrize("row", R.PAPER_TABLES)
def test_every_table_cell(row):
    dev, dse, so, fp, tx, t, oi_printed, perf_printed = row
    tol = 0.02 if (dev, dse, so) == ("v100", "aggressive", 8) else 0.01  # SPEC open question
    assert abs(R.operational_intensity(fp, tx) - oi_printed) <= tol
    rec = R.ProfileRecord(so, dse, fp, tx, t, 30000, 5)
    if not (dev == "v100" and dse == "basic"):  # Table 3 basic times duplicate Table 2
        assert abs(R.performance(rec) - perf_printed) <= 0.005 * perf_printed
    device = R.V100 if dev == "v100" else R.TITAN_Z
    assert R.classify(device, R.operational_intensity(fp, tx)) == "memory"  # PAPER §4


def test_performance_and_attainable_examples():
    assert abs(R.performance(R.ProfileRecord(8, "basic", 1450112268, 1, 553.92, 30000)) - 78.54) <= 0.05
    assert abs(R.performance(R.ProfileRecord(8, "aggressive", 641887345, 1, 135.73, 30000)) - 141.88) <= 0.05
    assert abs(R.performance(R.ProfileRecord(24, "aggressive", 929760267, 1, 18.48, 30000)) - 1509.60) <= 1.0
    assert abs(R.attainable_peak(R.V100, 2.49) - 2241) < 1
    assert abs(R.attainable_peak(R.TITAN_Z, 0.89) - 598.08) < 0.01
    assert abs(141.88 / R.attainable_peak(R.TITAN_Z, 0.89) - 0.237) < 0.001  # "24% of Titan Z"
    assert R.attainable_peak(R.V100, 1e6) == R.V100.sp_peak
    assert R.classify(R.V100, R.V100.ridge) == "compute"
    assert R.classify(R.V100, 100) == "compute"


def test_ingest_and_chart(tmp_path):
    text = ("space_order,dse,fp32_count,mem_transactions,total_time_s,timesteps,runs\n"
            "8,basic,1450112268,22722746,553.92,30000,5\n"
            '8,aggressive,"641,887,345","22,637,047","135,73",30000,5\n')
    recs = R.ingest_profiles(text)
    assert len(recs) == 2 and recs[1].total_time == 135.73 and recs[1].fp32_count == 641887345
    assert R.ingest_profiles("") == []
    with pytest.raises(ValueError, match="line 2"):
        R.ingest_profiles("space_order,dse\n8,basic,-1,2,3,4,5\n")
    pts = [R.point(R.TITAN_Z, r) for r in recs]
    svg, dat = R.emit_chart(pts, R.TITAN_Z)
    assert svg.startswith("<svg") and svg.count("<circle") == 2
    assert "so8_basic" in dat and dat.splitlines()[1].startswith("1.99")


def test_b200_point_is_memory_bound():
    rec = R.b200_record(8, "factorised", gpts=287.4, dram_bytes_per_point=17.3, flops_per_point=57)
    p = R.point(R.B200, rec)
    assert p.bound == "memory"
    assert abs(p.performance - 287.4 * 57) < 1
