"""The roofline models bench.py divides by (SURVEY §8(d) "Algorithmic work per circuit" table and
the streaming model), pinned to the table's printed figures: cfg3 per evaluation 3.54e9 FP64-pipe
ops and 8.32e9 on-chip bytes (t_FP64 0.190 ms, t_SMEM 0.224 ms at 148 SMs x 1.965 GHz), per-circuit
43,008 ops / 98,304 B (numerator) and 2,048 ops / 32,768 B (denominator) at n = 10, and the
streaming DRAM model (64N per numerator circuit while x is L2-resident, x added from n = 22, five
passes from n = 23).  CPU only."""

import numpy as np
import pytest

import bench
from dvqls_inputs import configs


def test_cfg3_models_match_survey_table():
    w = configs.cfg3()
    ops = bench.fp64_ops_per_eval(w)
    byts = bench.smem_bytes_per_eval(w)
    assert abs(ops - 3.54e9) / 3.54e9 < 0.005
    assert abs(byts - 8.32e9) / 8.32e9 < 0.005
    assert abs(ops / (64 * 148 * 1.965e9) * 1e3 - 0.190) < 0.001
    assert abs(byts / (128 * 148 * 1.965e9) * 1e3 - 0.224) < 0.001


def test_per_circuit_figures():
    w = configs.cfg3()
    num = np.array([2 * 1])           # circuit 2: task 1 = (l=0, k=0, s=1), a numerator
    den = np.array([0])               # circuit 0: task 0, s = 0, the denominator
    assert bench.fp64_ops_per_eval(w, num) == 43008
    assert bench.fp64_ops_per_eval(w, den) == 2048
    assert bench.smem_bytes_per_eval(w, num) == 98304
    assert bench.smem_bytes_per_eval(w, den) == 32768


@pytest.mark.parametrize("n", [16, 20, 22, 24])
def test_streaming_dram_model(n):
    w = configs.cfg5(n)
    N = 1 << n
    c = np.arange(w.n_circuits)
    s = (c // 2) % (n + 1)
    num, den = int(np.count_nonzero(s)), int(np.count_nonzero(s == 0))
    per_num = 64 if n <= 21 else (96 if n == 22 else 160)
    per_den = 0 if n <= 21 else 32
    assert bench.hbm_bytes_per_eval(w) == num * per_num * N + den * per_den * N
    # the SURVEY's 96N / 32N figure reported beside it (x counted as HBM at every n)
    assert bench.smem_bytes_per_eval(w) == num * 96 * N + den * 32 * N


def test_onchip_roofline_reports_the_binding_model():
    """cfg3: the SMEM model binds (0.224 vs 0.190 ms per evaluation), so bench.py reports
    bound = "smem" with frac = t_model / t_kernel and the FP64-pipe fraction beside it."""
    import numpy as np
    w = configs.cfg3()
    lc = np.arange(w.n_circuits)
    r = bench.onchip_roofline(w, lc, 16, 4.4, 148, 1965e6, "measured", "plane_kernel<20>")
    assert r["bound"] == "smem" and r["unit"] == "GB/s"
    assert abs(r["frac"] - r["model_frac"]) < 1e-12
    assert r["fp64"]["frac"] < r["frac"] and r["traffic"] is None


def test_parse_ncu_dram_csv():
    """roofline.traffic comes from an ncu CSV log of a --traffic-probe child (bench.measure_traffic):
    the parser finds the two DRAM metrics by the header's column names, skips ==PROF== lines and
    other metrics, keeps the first launch's values and survives thousands separators."""
    import csv
    import io
    log = (
        '==PROF== Connected to process 1\n'
        '"ID","Process ID","Process Name","Host Name","Kernel Name","Context","Stream","Block Size",'
        '"Grid Size","Device","CC","Section Name","Metric Name","Metric Unit","Metric Value"\n'
        '"0","1","python3","h","plane2_kernel","1","13","(384, 1, 1)","(148, 1, 1)","0","10.0",'
        '"Command line profiler metrics","dram__bytes_read.sum","byte","352,768"\n'
        '"0","1","python3","h","plane2_kernel","1","13","(384, 1, 1)","(148, 1, 1)","0","10.0",'
        '"Command line profiler metrics","dram__bytes_write.sum","byte","0"\n'
        '"0","1","python3","h","plane2_kernel","1","13","(384, 1, 1)","(148, 1, 1)","0","10.0",'
        '"Command line profiler metrics","gpu__time_duration.sum","nsecond","4300000"\n'
        '"1","1","python3","h","plane2_kernel","1","13","(384, 1, 1)","(148, 1, 1)","0","10.0",'
        '"Command line profiler metrics","dram__bytes_read.sum","byte","999"\n')
    vals = bench.parse_ncu_dram(list(csv.reader(io.StringIO(log))))
    assert vals == {"dram__bytes_read.sum": 352768.0, "dram__bytes_write.sum": 0.0}
    assert bench.parse_ncu_dram([["==PROF== nothing"]]) == {}
