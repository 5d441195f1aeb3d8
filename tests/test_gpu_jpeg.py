"""decode -> preprocess on the GPU: `io.decode_jpeg` (host entropy decoding
+ sm_100a IDCT / upsampling / colour kernels) against the reference
decoder's own outputs (tests/golden/jpeg.npz, bit-exact), the reference's
error classes, the batched path, and full-size frames against the oracle's
reconstruction (numpy, vectorised) of the same coefficients."""
import io as pyio
import os
import sys

import numpy as np
import pytest
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import jpeg_oracle as O  # noqa: E402

import paper_2505_12425_b200 as fv
import synth_fixtures  # noqa: E402
from paper_2505_12425_b200 import _native, synth  # noqa: E402
from paper_2505_12425_b200 import io as fio  # noqa: E402

pytestmark = pytest.mark.gpu

_Z = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "jpeg.npz"))
NAMES = sorted({k.split("__")[0] for k in _Z.files})
DECODED = [n for n in NAMES if n + "__out" in _Z.files]
REJECTED = [n for n in NAMES if n + "__err" in _Z.files]


def stream(name):
    return _Z[name + "__jpg"].tobytes()


@pytest.mark.parametrize("name", DECODED)
def test_matches_reference_decoder_exactly(name):
    out = fio.decode_jpeg(stream(name))
    assert out.is_cuda and out.dtype == torch.uint8
    assert np.array_equal(out.cpu().numpy(), _Z[name + "__out"])


@pytest.mark.parametrize("name", REJECTED)
def test_rejects_like_the_reference(name):
    ref = str(_Z[name + "__err"])
    cls = fv.UnsupportedJpegFeature if ref == "UnsupportedJpegFeature" else fv.CorruptStream
    with pytest.raises(cls):
        fio.decode_jpeg(stream(name))


@pytest.mark.parametrize("entropy", ["gpu", "host"])
def test_batch_matches_single(entropy):
    outs = fio.decode_jpeg_batch([stream(n) for n in DECODED], threads=8, entropy=entropy)
    for n, o in zip(DECODED, outs):
        assert np.array_equal(o.cpu().numpy(), _Z[n + "__out"]), n


def test_concurrent_batches_on_separate_streams():
    """Several host threads decoding batches at once, each on its own CUDA
    stream: the planner's worker pool, the pinned staging and the scratch
    pool are shared; every result must still be exact."""
    import threading
    names = DECODED
    data = [stream(n) for n in names]  # (the npz archive is read here: its lazy reader is not thread-safe)
    want = [_Z[n + "__out"] for n in names]
    errs = []

    def run(k):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for _ in range(4):
                    outs = fio.decode_jpeg_batch(data, threads=1 + k)
                    s.synchronize()
                    for n, o, w in zip(names, outs, want):
                        assert np.array_equal(o.cpu().numpy(), w), n
        except Exception as e:  # surfaced below
            errs.append(e)

    ts = [threading.Thread(target=run, args=(k,)) for k in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs


def test_batch_into_out_tensor():
    names = ["pil_ss0_q60", "pil_ss1_q85", "pil_ss2_q95"]  # same 77 x 129 x 3 frame
    out = torch.zeros((3, 77, 129, 3), dtype=torch.uint8, device="cuda")
    views = fio.decode_jpeg_batch([stream(n) for n in names], out=out)
    for i, n in enumerate(names):
        assert np.array_equal(out[i].cpu().numpy(), _Z[n + "__out"])
        assert views[i].data_ptr() == out[i].data_ptr()
    with pytest.raises(fv.ShapeMismatch):
        fio.decode_jpeg_batch([stream("pil_photo_256")], out=out[:1])


def test_gpu_entropy_path_really_runs():
    """Every valid golden stream (4:4:4 / 4:2:2 / 4:2:0 / 4:4:0, gray,
    restart markers, 16-bit tables, full-block noise at q100) is decoded by
    the GPU entropy path itself, not by the host fallback -- except the
    crafted one whose DC values exceed int16 (the GPU path's coefficient
    width), which must fall back and still match."""
    on_gpu = [n for n in DECODED if n != "asm_gray_dc_int16_overflow"]
    g0, h0 = fio.stats["gpu_entropy"], fio.stats["host_entropy"]
    outs = fio.decode_jpeg_batch([stream(n) for n in on_gpu], entropy="gpu")
    assert fio.stats["gpu_entropy"] - g0 == len(on_gpu)
    assert fio.stats["host_entropy"] == h0
    for n, o in zip(on_gpu, outs):
        assert np.array_equal(o.cpu().numpy(), _Z[n + "__out"]), n
    out = fio.decode_jpeg_batch([stream("asm_gray_dc_int16_overflow")], entropy="gpu")[0]
    assert fio.stats["host_entropy"] == h0 + 1
    assert np.array_equal(out.cpu().numpy(), _Z["asm_gray_dc_int16_overflow__out"])


@pytest.mark.parametrize("entropy", ["gpu", "host"])
def test_batch_raises_first_error(entropy):
    with pytest.raises(fv.CorruptStream):
        fio.decode_jpeg_batch([stream(DECODED[0]), stream("err_png")], entropy=entropy)
    with pytest.raises(fv.UnsupportedJpegFeature):  # header error vs entropy error: input order decides
        fio.decode_jpeg_batch([stream("err_progressive"), stream("fuzz_mut_03")], entropy=entropy)
    with pytest.raises(fv.CorruptStream):  # entropy error first
        fio.decode_jpeg_batch([stream("fuzz_mut_03"), stream("err_progressive")], entropy=entropy)
    # good streams after a header error are parsed but never written anywhere
    canary = torch.full((1 << 20,), 0x5A, dtype=torch.uint8, device="cuda")
    with pytest.raises(fv.CorruptStream):
        fio.decode_jpeg_batch([stream("pil_ss2_q85"), stream("err_png"), stream("pil_photo_256")], entropy=entropy)
    torch.cuda.synchronize()
    assert bool((canary == 0x5A).all())


@pytest.mark.parametrize("name", REJECTED)
def test_gpu_entropy_rejects_like_the_reference(name):
    """Every rejected golden stream, alone and behind a good one, through the
    GPU entropy path: same exception class as the reference."""
    ref = str(_Z[name + "__err"])
    cls = fv.UnsupportedJpegFeature if ref == "UnsupportedJpegFeature" else fv.CorruptStream
    with pytest.raises(cls):
        fio.decode_jpeg_batch([stream(name)], entropy="gpu")
    with pytest.raises(cls):
        fio.decode_jpeg_batch([stream("pil_photo_256"), stream(name)], entropy="gpu")


def test_gpu_entropy_fuzz_matches_host():
    """Byte mutations of a restart-marker stream and of a plain one: the GPU
    entropy path gives the host decoder's result (pixels or error class)."""
    rng = np.random.default_rng(91)
    for base_name in ("pil_restart_420", "pil_ss2_q85", "asm_440_q85"):
        base = stream(base_name)
        sos = base.find(b"\xff\xda")
        for _ in range(40):
            d = bytearray(base)
            for _ in range(int(rng.integers(1, 4))):
                d[int(rng.integers(sos + 14, len(d) - 2))] = int(rng.integers(0, 256))
            d = bytes(d)
            try:
                ref = fio.decode_jpeg(d).cpu().numpy()
            except fv.FoveaError as e:
                with pytest.raises(type(e)):
                    fio.decode_jpeg_batch([d], entropy="gpu")
                continue
            got = fio.decode_jpeg_batch([d], entropy="gpu")[0].cpu().numpy()
            assert np.array_equal(got, ref)


def test_batch_int16_overflow_image_and_repeats():
    """An image whose DC exceeds int16 inside a batch takes the int64 path;
    the others still come from the batched runtime; reusing the pinned
    staging across calls stays correct."""
    names = ["pil_photo_256", "asm_gray_dc_int16_overflow", "pil_ss2_q85", "asm_440_q85"]
    for _ in range(3):
        outs = fio.decode_jpeg_batch([stream(n) for n in names], threads=3)
        for n, o in zip(names, outs):
            assert np.array_equal(o.cpu().numpy(), _Z[n + "__out"]), n


def _pil(arr, **kw):
    from PIL import Image as PILImage
    b = pyio.BytesIO()
    PILImage.fromarray(arr).save(b, format="JPEG", **kw)
    return b.getvalue()


def _oracle_from_coefficients(data):
    """The oracle's reconstruction (vectorised numpy) of the library's host
    coefficients; the host entropy decoding is pinned against the oracle in
    tests/test_jpeg_host.py."""
    info, coef = fio.decode_coefficients(data)
    o = O.parse(data)
    comps = []
    for e, c in enumerate(o["comps"]):
        c["bw"], c["bh"] = info.bw[e], info.bh[e]
        comps.append(coef[info.coef_offset[e]:info.coef_offset[e] + 64 * c["bw"] * c["bh"]].reshape(-1, 64))
    planes = O.component_planes(o, comps)
    return planes[0].astype(np.uint8)[:, :, None] if len(planes) == 1 else O.ycbcr_to_rgb(*planes)


@pytest.mark.parametrize("sub", [0, 1, 2])
def test_full_frame_1080p(sub):
    pytest.importorskip("PIL")
    arr = synth.seeded_u8_image(1920, 1080, 3, seed=60 + sub)
    smooth = np.clip(arr.astype(np.int32) // 4 + 96, 0, 255).astype(np.uint8)  # milder spectrum
    data = _pil(smooth, quality=90, subsampling=sub)
    got = fio.decode_jpeg(data).cpu().numpy()
    assert np.array_equal(got, _oracle_from_coefficients(data))
    # the GPU entropy path on the same frame (no restart markers: one segment
    # of ~2000 self-synchronising subsequences), and with restart markers
    assert np.array_equal(fio.decode_jpeg_batch([data], entropy="gpu")[0].cpu().numpy(), got)
    data_rst = _pil(smooth, quality=90, subsampling=sub, restart_marker_blocks=5)
    got_rst = fio.decode_jpeg_batch([data_rst, data], entropy="gpu")
    assert np.array_equal(got_rst[0].cpu().numpy(), fio.decode_jpeg(data_rst).cpu().numpy())
    assert np.array_equal(got_rst[1].cpu().numpy(), got)


def test_gpu_entropy_smooth_and_noise_batch():
    """64 frames (smooth q90 4:2:0 like the bench, noise q95 4:4:4) through
    the GPU entropy path: identical to the single-image path."""
    pytest.importorskip("PIL")
    streams = []
    for i in range(6):
        streams.append(_pil(synth_fixtures.seeded_smooth_u8_image(640 + 16 * i, 360 + 8 * i, 3, seed=i), quality=90,
                            subsampling=2))
        streams.append(_pil(synth.seeded_u8_image(320 + i, 200 + 3 * i, 3, seed=i), quality=95, subsampling=0))
    outs = fio.decode_jpeg_batch(streams, entropy="gpu")
    for d, o in zip(streams, outs):
        assert np.array_equal(o.cpu().numpy(), fio.decode_jpeg(d).cpu().numpy())


def test_odd_sizes_restart_and_gray_full_path():
    pytest.importorskip("PIL")
    rng = np.random.default_rng(5)
    for (w, h, sub, rst) in [(1001, 777, 2, 0), (641, 479, 1, 7), (333, 1, 2, 0), (1, 333, 2, 3)]:
        arr = rng.integers(0, 256, (h, w, 3), dtype=np.uint8)
        kw = {"restart_marker_blocks": rst} if rst else {}
        data = _pil(arr, quality=85, subsampling=sub, **kw)
        assert np.array_equal(fio.decode_jpeg(data).cpu().numpy(), _oracle_from_coefficients(data)), (w, h)
    g = rng.integers(0, 256, (123, 457), dtype=np.uint8)
    data = _pil(g, quality=75)
    out = fio.decode_jpeg(data).cpu().numpy()
    assert out.shape == (123, 457, 1)
    assert np.array_equal(out, _oracle_from_coefficients(data))


def test_deterministic_and_native():
    n0 = _native.lib().fv_launch_count()
    a = fio.decode_jpeg(stream("pil_photo_256"))
    b = fio.decode_jpeg(stream("pil_photo_256"))
    torch.cuda.synchronize()
    assert torch.equal(a, b)
    assert _native.lib().fv_launch_count() - n0 == 4  # IDCT + colour kernels per decode


def test_decode_then_preprocess():
    """The chain the row is named for: decoded frame -> fused resize ->
    normalise -> CHW, against the oracle on the same decoded pixels."""
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
    import fovea_oracle as FO
    img = fio.decode_jpeg(stream("pil_photo_256"))
    dst = torch.empty((3, 96, 128), dtype=torch.float32, device=img.device)
    fv.resize_normalize_chw(img, dst, synth.MEAN, synth.STD)
    ref = FO.resize_normalize_chw(_Z["pil_photo_256__out"], 128, 96, synth.MEAN, synth.STD)
    assert np.array_equal(dst.cpu().numpy(), ref)


@pytest.mark.parametrize("name", ["pil_photo_256", "pil_ss2_q85", "asm_440_q85", "pil_ss1_q85", "ref_gray_q92",
                                  "pil_odd_33x31"])
@pytest.mark.parametrize("width", [2, 8])
def test_reconstruct_crafted_coefficients(name, width):
    """Dequantisation + IDCT + upsampling + colour of crafted coefficients --
    mostly small blocks, some blocks over the full int16 range, 8- and 16-bit
    quantisers -- so that both IDCT passes take their int32 and their int64
    branches (a warp-uniform choice in the batch kernel); int16 input goes
    through the batch kernels, int64 input through the dense kernel; both
    against the oracle's int64 arithmetic (jpeg.py:163-203)."""
    data = stream(name)
    info = fio.jpeg_info(data)
    rng = np.random.default_rng(11 + width)
    nblk = info.coef_count // 64
    coef = rng.integers(-40, 41, (nblk, 64))
    wild = rng.random(nblk) < 0.08
    coef[wild] = rng.integers(-32768, 32768, (int(wild.sum()), 64))
    coef = coef.reshape(-1)
    hi = [255, 65535, 16]
    for e in range(info.ncomp):
        q = rng.integers(1, hi[e] + 1, 64)
        for k in range(64):
            info.qt[e][k] = int(q[k])
    o = O.parse(data)
    comps = []
    for e, c in enumerate(o["comps"]):
        c["bw"], c["bh"] = info.bw[e], info.bh[e]
        c["q"] = np.array([info.qt[e][k] for k in range(64)], np.int64)
        comps.append(coef[info.coef_offset[e]:info.coef_offset[e] + 64 * c["bw"] * c["bh"]].reshape(-1, 64))
    planes = O.component_planes(o, comps)
    ref = planes[0].astype(np.uint8)[:, :, None] if len(planes) == 1 else O.ycbcr_to_rgb(*planes)
    host = torch.from_numpy(coef.astype(np.int16 if width == 2 else np.int64))
    got = fio._reconstruct(info, host, width, torch.device("cuda", 0))
    torch.cuda.synchronize()
    assert np.array_equal(got.cpu().numpy(), ref)
