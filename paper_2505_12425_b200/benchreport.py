"""GPU benchmark harness with the reference's `BenchReport` wire format.

Mirror of `fovea.bench` (bench.py:31-192) for the B200 path (SURVEY §8(f)
rank 2): the same `run_benchmark(op, size, iterations, warmup) -> BenchReport`
call, the same report fields and invariants (bench.py:31-49), the same
JSON/CSV rendering (bench.py:167-192), the same per-op seeded fixtures
(bench.py:59-86: seeds 11-15, 2x up-scaling for the resizes), and the same
zero-allocation guard over the timed loop -- enforced here with the CUDA
caching allocator's allocation counter instead of `CountingAllocator`.

Differences, all additive: iterations are timed with CUDA events on the
launching stream (not `perf_counter_ns`), the report carries `gbs`
(algorithmic bytes / mean time) and `device`, and the op registry adds the
path's new ops (u8 bilinear, warps, fused preprocessing). Codec ops
(decode_png, decode_jpeg, encode_jpeg) are outside the GPU path and raise
`UnknownOp`, as any unregistered op does.
"""
from __future__ import annotations

import csv
import io
import json
import sys
from dataclasses import asdict, dataclass, fields
from datetime import datetime, timezone

import numpy as np
import torch

from . import imgproc
from .errors import FoveaError
from . import synth


class UnknownOp(FoveaError):
    """Benchmark operation name not in the registry (errors.py:126-127)."""


class FixtureFailure(FoveaError):
    """Benchmark fixture could not be constructed (errors.py:130-131)."""


@dataclass
class BenchReport:
    """bench.py:31-49, plus `gbs` and `device`."""

    op: str
    width: int
    height: int
    iterations: int
    mean_ns: float
    median_ns: float
    p95_ns: float
    stddev_ns: float
    throughput_megapixels_per_s: float | None
    timestamp: str
    profile: str
    gbs: float | None = None
    device: str = ""

    def __post_init__(self):
        if self.iterations < 1:
            raise FixtureFailure("iterations must be >= 1")
        if not (self.median_ns <= self.p95_ns and self.mean_ns > 0 and self.median_ns > 0):
            raise FixtureFailure("inconsistent timing aggregates")


def _profile() -> str:
    return f"cuda-{torch.version.cuda}-torch-{torch.__version__}-sm_100a"


def _u8(w, h, c, seed, dev):
    return torch.from_numpy(synth.seeded_u8_image(w, h, c, seed)).to(dev)


def _f32(w, h, c, seed, dev):
    return torch.from_numpy(synth.seeded_f32_image(w, h, c, seed)).to(dev)


# op -> setup(size, dev) -> (run, algorithmic bytes per run); seeds as bench.py:59-86
def _gray(size, dev):
    src = _u8(size.width, size.height, 3, 11, dev)
    dst = torch.zeros((size.height, size.width, 1), dtype=torch.uint8, device=dev)
    return (lambda: imgproc.gray_from_rgb(src, dst)), src.numel() + dst.numel()


def _flip(size, dev):
    src = _u8(size.width, size.height, 3, 12, dev)
    dst = torch.zeros_like(src)
    return (lambda: imgproc.flip_horizontal(src, dst)), 2 * src.numel()


def _nearest(size, dev):
    src = _u8(size.width, size.height, 3, 13, dev)
    dst = torch.zeros((2 * size.height, 2 * size.width, 3), dtype=torch.uint8, device=dev)
    return (lambda: imgproc.resize_nearest(src, dst)), src.numel() + dst.numel()


def _bilinear(size, dev):
    src = _f32(size.width, size.height, 3, 14, dev)
    dst = torch.zeros((2 * size.height, 2 * size.width, 3), dtype=torch.float32, device=dev)
    return (lambda: imgproc.resize_bilinear(src, dst)), 4 * (src.numel() + dst.numel())


def _sobel(size, dev):
    src = _f32(size.width, size.height, 3, 15, dev)
    dst = torch.zeros_like(src)
    return (lambda: imgproc.sobel(src, dst, 3)), 8 * src.numel()


def _bilinear_u8(size, dev):
    src = _u8(size.width, size.height, 3, 14, dev)
    dst = torch.zeros((2 * size.height, 2 * size.width, 3), dtype=torch.uint8, device=dev)
    return (lambda: imgproc.resize_bilinear_u8(src, dst)), src.numel() + dst.numel()


def _affine(size, dev):
    src = _f32(size.width, size.height, 3, 30000, dev)
    dst = torch.zeros_like(src)
    m = synth.affine_forward(31000, size.width, size.height)
    return (lambda: imgproc.warp_affine(src, dst, m)), 8 * src.numel()


def _perspective(size, dev):
    src = _u8(size.width, size.height, 3, 40000, dev)
    dst = torch.zeros_like(src)
    hm = synth.perspective_forward(41000)
    return (lambda: imgproc.warp_perspective(src, dst, hm)), 2 * src.numel()


def _fused(size, dev):
    src = _u8(size.width, size.height, 3, 50000, dev)
    dst = torch.zeros((3, 640, 640), dtype=torch.float32, device=dev)
    return (lambda: imgproc.resize_normalize_chw(src, dst, synth.MEAN, synth.STD)), src.numel() + 4 * dst.numel()


_OPS = {
    "gray_from_rgb": _gray,
    "flip_horizontal": _flip,
    "resize_nearest": _nearest,
    "resize_bilinear": _bilinear,
    "sobel": _sobel,
    "resize_bilinear_u8": _bilinear_u8,
    "warp_affine": _affine,
    "warp_perspective": _perspective,
    "resize_normalize_chw": _fused,
}

OP_NAMES = tuple(_OPS)


@dataclass(frozen=True)
class Size:
    width: int
    height: int


def run_benchmark(op: str, size, iterations: int, warmup: int = 5, device="cuda") -> BenchReport:
    """bench.py:118-164 on the GPU: warm up, time `iterations` runs with CUDA
    events, assert the timed loop allocated no device memory."""
    if op not in _OPS:
        raise UnknownOp(f"unknown op {op!r}; expected one of {', '.join(OP_NAMES)}")
    if iterations < 1:
        raise FixtureFailure("iterations must be >= 1")
    if warmup < 0:
        raise FixtureFailure("warmup must be >= 0")
    dev = torch.device(device)
    try:
        run, nbytes = _OPS[op](size, dev)
    except FoveaError:
        raise
    except Exception as e:
        raise FixtureFailure(f"cannot build fixture for {op} at {size.width}x{size.height}: {e}") from e
    for _ in range(warmup):
        run()
    torch.cuda.synchronize(dev)
    stream = torch.cuda.current_stream(dev)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iterations)]
    allocs_before = torch.cuda.memory_stats(dev).get("allocation.all.allocated", 0)
    for a, b in ev:
        a.record(stream)
        run()
        b.record(stream)
    torch.cuda.synchronize(dev)
    if torch.cuda.memory_stats(dev).get("allocation.all.allocated", 0) != allocs_before:
        raise FixtureFailure(f"{op} allocated device memory during the timed loop")
    times = np.array([a.elapsed_time(b) * 1e6 for a, b in ev], dtype=np.float64)  # ns
    total_s = float(times.sum()) / 1e9
    pixels = size.width * size.height * iterations  # source pixels, bench.py:151
    return BenchReport(
        op=op, width=size.width, height=size.height, iterations=iterations,
        mean_ns=float(times.mean()), median_ns=float(np.median(times)), p95_ns=float(np.percentile(times, 95)),
        stddev_ns=float(times.std()), throughput_megapixels_per_s=pixels / total_s / 1e6,
        timestamp=datetime.now(timezone.utc).isoformat(timespec="seconds"), profile=_profile(),
        gbs=nbytes / (float(times.mean()) / 1e9) / 1e9, device=torch.cuda.get_device_name(dev),
    )


def render_report(reports: list, fmt: str = "json") -> str:
    """bench.py:167-179."""
    if fmt == "json":
        return json.dumps([asdict(r) for r in reports], indent=2)
    if fmt == "csv":
        names = [f.name for f in fields(BenchReport)]
        buf = io.StringIO()
        writer = csv.DictWriter(buf, fieldnames=names, lineterminator="\n")
        writer.writeheader()
        for r in reports:
            writer.writerow(asdict(r))
        return buf.getvalue()
    raise FoveaError(f"unknown report format {fmt!r}")


def emit_report(reports: list, fmt: str = "json", path=None) -> None:
    """bench.py:182-192."""
    text = render_report(reports, fmt)
    if path is None:
        sys.stdout.write(text + ("" if text.endswith("\n") else "\n"))
        return
    with open(path, "w", encoding="utf-8") as f:
        f.write(text + ("" if text.endswith("\n") else "\n"))


def main(argv=None) -> int:
    """`python -m paper_2505_12425_b200.benchreport --op OP --width W --height H
    --iters N [--warmup K] [--format json|csv]` (the reference CLI's `bench`,
    cli.py:66-80, run in process)."""
    import argparse

    ap = argparse.ArgumentParser(prog="fovea-b200-bench")
    ap.add_argument("--op", required=True)
    ap.add_argument("--width", type=int, default=1920)
    ap.add_argument("--height", type=int, default=1080)
    ap.add_argument("--iters", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--format", default="json", choices=["json", "csv"])
    a = ap.parse_args(argv)
    try:
        emit_report([run_benchmark(a.op, Size(a.width, a.height), a.iters, a.warmup)], a.format)
    except FoveaError as e:
        sys.stderr.write(f"error: {type(e).__name__}: {e}\n")
        return 2
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
