"""BenchReport wire format (reference bench.py:31-192 / test_bench.py),
CPU parts here, GPU runs marked."""
import csv
import io
import json

import pytest

from paper_2505_12425_b200 import benchreport as br


def _report(**kw):
    base = dict(op="gray_from_rgb", width=8, height=8, iterations=3, mean_ns=10.0, median_ns=9.0, p95_ns=12.0,
                stddev_ns=1.0, throughput_megapixels_per_s=1.0, timestamp="t", profile="p")
    base.update(kw)
    return br.BenchReport(**base)


def test_unknown_op_and_codecs_are_not_gpu_ops():
    for op in ("warp_something", "decode_png", "decode_jpeg", "encode_jpeg"):
        with pytest.raises(br.UnknownOp):
            br.run_benchmark(op, br.Size(8, 8), 1)


def test_bad_iterations_rejected():
    with pytest.raises(br.FixtureFailure):
        br.run_benchmark("gray_from_rgb", br.Size(8, 8), 0)
    with pytest.raises(br.FixtureFailure):
        _report(iterations=0)
    with pytest.raises(br.FixtureFailure):
        _report(median_ns=20.0, p95_ns=12.0)


def test_render_json_and_csv_schema():
    reps = [_report(), _report(op="sobel")]
    js = json.loads(br.render_report(reps, "json"))
    assert [r["op"] for r in js] == ["gray_from_rgb", "sobel"]
    rows = list(csv.DictReader(io.StringIO(br.render_report(reps, "csv"))))
    ref_fields = ["op", "width", "height", "iterations", "mean_ns", "median_ns", "p95_ns", "stddev_ns",
                  "throughput_megapixels_per_s", "timestamp", "profile"]
    assert list(rows[0].keys())[: len(ref_fields)] == ref_fields  # the reference's columns first
    with pytest.raises(br.FoveaError):
        br.render_report(reps, "xml")


@pytest.mark.gpu
@pytest.mark.parametrize("op", br.OP_NAMES)
def test_every_op_runs_on_gpu(op):
    r = br.run_benchmark(op, br.Size(64, 48), iterations=2, warmup=1)
    assert r.op == op and r.median_ns <= r.p95_ns and r.gbs > 0


@pytest.mark.gpu
def test_single_iteration_degenerate_stats_and_throughput():
    r = br.run_benchmark("gray_from_rgb", br.Size(32, 32), iterations=1, warmup=1)
    assert r.mean_ns == r.median_ns == r.p95_ns and r.stddev_ns == 0.0
    r = br.run_benchmark("gray_from_rgb", br.Size(128, 128), iterations=25, warmup=2)
    assert r.throughput_megapixels_per_s == pytest.approx(128 * 128 * 25 / (r.mean_ns * 25 / 1e9) / 1e6, rel=1e-9)


@pytest.mark.gpu
def test_cli_json(capsys):
    assert br.main(["--op", "resize_bilinear_u8", "--width", "256", "--height", "128", "--iters", "5"]) == 0
    out = json.loads(capsys.readouterr().out)
    assert out[0]["op"] == "resize_bilinear_u8"
    assert br.main(["--op", "decode_png", "--iters", "1"]) == 2
