"""decode -> preprocess, host side (no GPU): the oracle against the
reference's own outputs, and the C ABI's header parsing + entropy decoding
against the oracle -- coefficients bit-identical, errors of the same class.

The GPU reconstruction is covered by tests/test_gpu_jpeg.py."""
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import jpeg_oracle as O  # noqa: E402

import paper_2505_12425_b200 as fv  # noqa: E402
from paper_2505_12425_b200 import io as fio  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "jpeg.npz")
_Z = np.load(GOLDEN)
NAMES = sorted({k.split("__")[0] for k in _Z.files})
FOVEA_ERRORS = ("CorruptStream", "UnsupportedJpegFeature")


def stream(name):
    return _Z[name + "__jpg"].tobytes()


def expected_error(name):
    """The reference's exception class; its non-FoveaError failures (e.g.
    IndexError on an overfull Huffman table) are CorruptStream here."""
    e = str(_Z[name + "__err"])
    return e if e in FOVEA_ERRORS else "CorruptStream"


def oracle_outcome(data):
    try:
        info = O.parse(data)
        return info, O.decode_coefficients(info), None
    except (O.CorruptStream, O.UnsupportedJpegFeature) as e:
        return None, None, type(e).__name__


def ours(data):
    try:
        info, coef = fio.decode_coefficients(data)
        return info, coef, None
    except (fv.CorruptStream, fv.UnsupportedJpegFeature) as e:
        return None, None, type(e).__name__


def assert_same(data):
    oi, oc, oe = oracle_outcome(data)
    info, coef, err = ours(data)
    assert err == oe, f"error class {err} != oracle {oe}"
    if oe is not None:
        return
    assert (info.width, info.height, info.ncomp) == (oi["width"], oi["height"], len(oi["comps"]))
    assert info.restart_interval == oi["dri"]
    for e, c in enumerate(oi["comps"]):
        assert (info.h[e], info.v[e], info.bw[e], info.bh[e]) == (c["h"], c["v"], c["bw"], c["bh"])
        n = c["bw"] * c["bh"] * 64
        got = coef[info.coef_offset[e]:info.coef_offset[e] + n].reshape(-1, 64)
        assert np.array_equal(got, oc[e]), f"component {e} coefficients differ"
        assert np.array_equal(np.array(info.qt[e][:], np.int64), c["q"])


@pytest.mark.parametrize("name", NAMES)
def test_oracle_matches_reference(name):
    data = stream(name)
    if name + "__out" in _Z.files:
        assert np.array_equal(O.decode_jpeg(data), _Z[name + "__out"])
    else:
        with pytest.raises((O.CorruptStream, O.UnsupportedJpegFeature)) as ei:
            O.decode_jpeg(data)
        assert type(ei.value).__name__ == expected_error(name)


@pytest.mark.parametrize("name", NAMES)
def test_host_decoder_matches_oracle(name):
    assert_same(stream(name))


def test_fuzzed_mutations_agree_and_never_crash():
    """jpeg test_fuzzed_mutations_never_crash, made stricter: every mutated
    stream gets the oracle's outcome (same coefficients or same error)."""
    base = stream("ref444_q90")
    rng = np.random.default_rng(77)
    for _ in range(150):
        d = bytearray(base)
        for _ in range(int(rng.integers(1, 6))):
            d[int(rng.integers(0, len(d)))] = int(rng.integers(0, 256))
        assert_same(bytes(d))


def test_fuzzed_truncations_agree():
    base = stream("pil_restart_420")
    for cut in np.random.default_rng(78).integers(0, len(base), size=60):
        assert_same(base[:int(cut)])


def test_header_mutations_agree():
    """Mutations confined to the headers (tables, SOF, SOS, DRI): the
    decoder's checks, in the reference's order."""
    base = stream("asm_420_q16_rst")
    sos = base.find(b"\xff\xda")
    rng = np.random.default_rng(79)
    for _ in range(150):
        d = bytearray(base)
        for _ in range(int(rng.integers(1, 4))):
            d[int(rng.integers(2, sos + 14))] = int(rng.integers(0, 256))
        assert_same(bytes(d))


def test_implausible_header_rejected_before_allocation():
    """A frame header claiming 65535 x 65535 pixels over a tiny scan is
    corrupt (each block needs >= 2 bits); it is rejected by the header pass,
    not after allocating gigabytes of coefficients."""
    d = bytearray(stream("ref444_q90"))
    i = d.find(b"\xff\xc0")
    d[i + 5:i + 9] = b"\xff\xff\xff\xff"
    with pytest.raises(fv.CorruptStream):
        fio.jpeg_info(bytes(d))


def test_not_bytes_rejected():
    with pytest.raises(fv.CorruptStream):
        fio.jpeg_info("not bytes")


def _info_batch(streams, threads):
    import ctypes
    from paper_2505_12425_b200 import _native
    n = len(streams)
    data = (ctypes.c_char_p * n)(*streams)
    lens = (ctypes.c_int64 * n)(*[len(b) for b in streams])
    infos = (_native.FvJpegInfo * n)()
    status = (ctypes.c_int32 * n)()
    assert _native.lib().fv_jpeg_info_batch(data, lens, n, infos, status, threads) == 0
    return [(status[i], infos[i].width, infos[i].height, infos[i].ncomp, infos[i].coef_count) for i in range(n)]


def test_worker_pool_concurrent_batches():
    """The batch entry points share one persistent worker pool: concurrent
    callers (ctypes drops the GIL) each get their own complete results."""
    import threading
    streams = [stream(n) for n in NAMES] * 4
    want = _info_batch(streams, 1)
    assert any(s == 0 for s, *_ in want) and any(s != 0 for s, *_ in want)
    got, errs = {}, []

    def run(k):
        try:
            for _ in range(20):
                got[k] = _info_batch(streams, 1 + k % 5)
                assert got[k] == want
        except Exception as e:  # surfaced below
            errs.append(e)

    ts = [threading.Thread(target=run, args=(k,)) for k in range(6)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    assert len(got) == 6


@pytest.mark.skipif(not hasattr(os, "fork"), reason="fork")
@pytest.mark.filterwarnings("ignore::DeprecationWarning")  # forking a multi-threaded process is the point
def test_worker_pool_after_fork():
    """A forked child (data-loader workers) gets a fresh pool: the parent's
    threads do not exist there."""
    streams = [stream(n) for n in NAMES]
    want = _info_batch(streams, 4)  # the parent's pool exists now
    pid = os.fork()
    if pid == 0:  # child: must finish, and agree
        try:
            code = 0 if _info_batch(streams, 4) == want else 3
        except BaseException:
            code = 4
        os._exit(code)
    _, st = os.waitpid(pid, 0)
    assert os.WIFEXITED(st) and os.WEXITSTATUS(st) == 0
