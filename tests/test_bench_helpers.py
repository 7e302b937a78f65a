"""bench.py's host-side report helpers (no GPU): the reference CSV schema
(SimMetrics::csv_header / csv_row, /root/reference/proj/src/sim.cpp:58-70,
format_double = std::to_chars shortest round trip, util.hpp:45-49) and the
algorithmic-bytes model of step_roofline."""
import importlib.util
import os

import vc_testlib as T

spec = importlib.util.spec_from_file_location("bench", os.path.join(T.ROOT, "bench.py"))
bench = importlib.util.module_from_spec(spec)
spec.loader.exec_module(bench)


def test_csv_header_is_the_reference_schema():
    ref = open("/root/reference/proj/src/sim.cpp").read() if os.path.exists("/root/reference/proj/src/sim.cpp") else None
    assert bench.CSV_HEADER == ("schedule,B,x,c,throughput_tok_s,p50_latency_s,p99_latency_s,peak_hbm_bytes,"
                                "interconnect_busy")
    if ref:
        assert '"schedule,B,x,c,throughput_tok_s,p50_latency_s,p99_latency_s,peak_hbm_bytes,"' in ref


def test_format_double_shortest_round_trip():
    assert bench.fmt_double(5.0) == "5"
    assert bench.fmt_double(0.1) == "0.1"
    assert bench.fmt_double(1474.8) == "1474.8"
    assert bench.fmt_double(1e-05) == "1e-05"
    assert bench.csv_row("staggered", 16, 6, 0.25, 1474.8, 0.0, 0.0, 123, 0.5) == \
        "staggered,16,6,0.25,1474.8,0,0,123,0.5"


def test_step_roofline_bytes_model():
    from paper_2605_17613_b200 import LLAMA3_8B
    w = bench.weight_read_bytes(LLAMA3_8B)
    assert 14.9e9 < w < 15.1e9  # 32 layers of projections + the LM head
    r = {"x": 6, "meta": {"full_bytes": 4_294_967_296, "payload_bytes": 1_073_741_824, "aux_bytes": 67_108_864},
         "st": {"timed_iterations": 10, "timed_verifies": 20, "timed_rows": 10 * 14 + 20 * 7,
                "timed_verify_rows": 140, "timed_device_ms": 90.0}}
    out = bench.step_roofline(r, LLAMA3_8B, 6547.5)
    want = 10 * w + 140 * (1_073_741_824 + 67_108_864) + 20 * 4_294_967_296
    assert out["bytes_per_iteration"] == int(want / 10)
    assert abs(out["achieved_gbs"] - want / 0.09 / 1e9) < 0.1


def test_sim_metrics_null_latency_without_completions():
    base = {"throughput": 10.0, "warm_throughput": 11.0, "interconnect_busy": 0.5, "peak_hbm_bytes": 7}
    m = bench.sim_metrics(dict(base, p50_latency_s=0.0, p99_latency_s=0.0))
    assert m["p50_latency_s"] is None and m["p99_latency_s"] is None and "latency_note" in m
    m = bench.sim_metrics(dict(base, p50_latency_s=1.5, p99_latency_s=2.25))
    assert m["p50_latency_s"] == 1.5 and m["p99_latency_s"] == 2.25 and "latency_note" not in m
