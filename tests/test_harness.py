"""Dataset harness, on-disk formats and image metrics.

The B200 harness (csrc/harness.cpp: device-batched press episodes, host
writer pool) is compared with the reference's own dataset::run_press_dataset
(harness.cpp:159-245) on tests/scenes.HARNESS: tests/golden/harness.npz holds
its manifest.csv, config.json, every image and .depth file, and
metrics::compare (image_metrics.cpp:57-112) on image pairs
(tests/golden/make_golden.py::harness).

Tolerances: manifest and config.json byte-identical; images <= 2/255 and
depth <= 1e-7 m (the capture bar of tests/test_gpu_parity.py); PSNR and MAE
exact (integer sums); SSIM <= 1e-10 (direct window sums on the GPU versus the
reference's summed-area tables).
"""
import json
import os
import shutil
import struct
import zlib

import numpy as np
import pytest

from tests.scenes import HARNESS

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def golden():
    return np.load(os.path.join(ROOT, "tests", "golden", "harness.npz"))


def _tb():
    import paper_2301_08343_b200 as tb

    return tb


# ---- PNG codec (CPU) ---------------------------------------------------------


def _png(path, w, h, ctype, depth, rows, plte=None, filters=None):
    """Minimal PNG encoder used to feed the decoder every filter type."""
    ch = {0: 1, 2: 3, 3: 1, 4: 2, 6: 4}[ctype]
    bpp = max(1, ch * depth // 8)
    raw = b""
    prev = bytearray(len(rows[0]))
    for r, line in enumerate(rows):
        ft = filters[r % len(filters)] if filters else 0
        out = bytearray(len(line))
        for i, x in enumerate(line):
            a = line[i - bpp] if i >= bpp else 0
            b = prev[i]
            c = prev[i - bpp] if i >= bpp else 0
            if ft == 0:
                p = 0
            elif ft == 1:
                p = a
            elif ft == 2:
                p = b
            elif ft == 3:
                p = (a + b) // 2
            else:
                pa, pb, pc = abs(b - c), abs(a - c), abs(a + b - 2 * c)
                p = a if pa <= pb and pa <= pc else (b if pb <= pc else c)
            out[i] = (x - p) & 255
        raw += bytes([ft]) + bytes(out)
        prev = bytearray(line)

    def chunk(t, body):
        return struct.pack(">I", len(body)) + t + body + struct.pack(">I", zlib.crc32(t + body))

    data = b"\x89PNG\r\n\x1a\n" + chunk(b"IHDR", struct.pack(">IIBBBBB", w, h, depth, ctype, 0, 0, 0))
    if plte is not None:
        data += chunk(b"PLTE", bytes(plte))
    data += chunk(b"IDAT", zlib.compress(raw)) + chunk(b"IEND", b"")
    with open(path, "wb") as f:
        f.write(data)


def test_png_roundtrip(tmp_path):
    tb = _tb()
    img = np.random.default_rng(0).integers(0, 256, (23, 31, 3), dtype=np.uint8)
    tb.save_png(img, str(tmp_path / "a.png"))
    np.testing.assert_array_equal(tb.load_png(str(tmp_path / "a.png")), img)


def test_png_decoder_filters_and_colour_types(tmp_path):
    """load_png's expansion rules (image.cpp:71-75): palette / grey expanded,
    16-bit stripped to the high byte, alpha dropped; all five filters."""
    tb = _tb()
    rng = np.random.default_rng(1)
    h, w = 9, 11
    rgb = rng.integers(0, 256, (h, w, 3), dtype=np.uint8)
    p = str(tmp_path / "f.png")
    _png(p, w, h, 2, 8, [bytes(r.ravel()) for r in rgb], filters=[0, 1, 2, 3, 4])
    np.testing.assert_array_equal(tb.load_png(p), rgb)
    rgba = np.concatenate([rgb, rng.integers(0, 256, (h, w, 1), dtype=np.uint8)], axis=2)
    _png(p, w, h, 6, 8, [bytes(r.ravel()) for r in rgba], filters=[4, 3, 1])
    np.testing.assert_array_equal(tb.load_png(p), rgb)
    grey = rng.integers(0, 256, (h, w), dtype=np.uint8)
    _png(p, w, h, 0, 8, [bytes(r) for r in grey], filters=[2, 4])
    np.testing.assert_array_equal(tb.load_png(p), np.repeat(grey[:, :, None], 3, axis=2))
    rgb16 = rng.integers(0, 65536, (h, w, 3), dtype=np.uint16)
    _png(p, w, h, 2, 16, [rr.astype(">u2").tobytes() for rr in rgb16], filters=[1, 4])
    np.testing.assert_array_equal(tb.load_png(p), (rgb16 >> 8).astype(np.uint8))
    pal = rng.integers(0, 256, (16, 3), dtype=np.uint8)
    idx = rng.integers(0, 16, (h, w), dtype=np.uint8)
    _png(p, w, h, 3, 8, [bytes(r) for r in idx], plte=pal.ravel(), filters=[0, 3])
    np.testing.assert_array_equal(tb.load_png(p), pal[idx])
    with open(p, "wb") as f:
        f.write(b"not a png")
    with pytest.raises(tb.ParseError):
        tb.load_png(p)
    with pytest.raises(tb.IoError):
        tb.load_png(str(tmp_path / "missing.png"))


# ---- harness host logic (CPU) ---------------------------------------------------


def test_config_json_matches_reference(golden, tmp_path):
    """config.json is written before any device work (harness.cpp:162):
    to_json_string (scene_config.cpp:124-170) byte-identical. Without a GPU the
    run then fails loudly (no CPU fallback)."""
    tb = _tb()
    try:
        tb.dataset.run_press_dataset(HARNESS, str(tmp_path))
        ran = True
    except tb.CudaError:
        ran = False
    with open(tmp_path / "config.json") as f:
        assert f.read() == str(golden["config_json"])
    assert os.path.isdir(tmp_path / "images") and os.path.isdir(tmp_path / "depth")
    if not ran:
        assert not os.path.exists(tmp_path / "manifest.csv")


def test_invalid_config_is_rejected(tmp_path):
    tb = _tb()
    with pytest.raises(tb.ConfigError, match="press.depths_mm must not be empty"):
        tb.dataset.run_press_dataset({**HARNESS, "press_grid": {"depths_mm": []}}, str(tmp_path))


def _write_manifest(d, rows):
    os.makedirs(d, exist_ok=True)
    with open(os.path.join(d, "manifest.csv"), "w") as f:
        f.write("object,position_index,pos_x_mm,pos_y_mm,depth_index,depth_mm,contact,"
                "particle_count,image,depth_map\n")
        for o, p, k in rows:
            f.write(f"{o},{p},0,0,{k},0,0,1,images/x.png,depth/x.depth\n")


def test_compare_datasets_manifest_mismatch(tmp_path):
    """compare_datasets checks the key sets before reading any image
    (harness.cpp:252-276)."""
    tb = _tb()
    a, b = str(tmp_path / "a"), str(tmp_path / "b")
    _write_manifest(a, [("sphere", 0, 0), ("sphere", 0, 1)])
    _write_manifest(b, [("sphere", 0, 0), ("dots", 3, 2)])
    with pytest.raises(tb.ManifestMismatch) as e:
        tb.dataset.compare_datasets(a, b)
    assert str(e.value) == ("manifests differ (2 keys): sphere/p0/d1 missing in B; "
                            "dots/p3/d2 missing in A")
    with open(os.path.join(b, "manifest.csv"), "a") as f:
        f.write("bad,row\n")
    with pytest.raises(tb.ParseError):
        tb.dataset.compare_datasets(a, b)


# ---- device path ------------------------------------------------------------------


def _split_depth(raw):
    raw = bytes(raw)
    nl = raw.index(b"\n")
    return raw[:nl], np.frombuffer(raw[nl + 1:], dtype=np.float32)


def _check_against_golden(tb, golden, d):
    with open(os.path.join(d, "manifest.csv")) as f:
        manifest = f.read()
    assert manifest == str(golden["manifest"])
    for line in manifest.splitlines()[1:]:
        f = line.split(",")
        key = f"{f[0]}_p{int(f[1])}_d{int(f[4])}"
        img = tb.load_png(os.path.join(d, f[8]))
        assert np.abs(img.astype(int) - golden[f"image_{key}"]).max() <= 2, key
        with open(os.path.join(d, f[9]), "rb") as fh:
            head, vals = _split_depth(fh.read())
        ghead, gvals = _split_depth(golden[f"depth_{key}"])
        assert head == ghead
        np.testing.assert_allclose(vals, gvals, rtol=0, atol=1e-7)


@pytest.mark.gpu
def test_press_dataset_matches_reference(golden, tmp_path):
    tb = _tb()
    d = str(tmp_path / "ds")
    rows, skipped = tb.dataset.run_press_dataset(HARNESS, d)
    assert (rows, skipped) == (int(golden["rows"]), int(golden["skipped"]))
    _check_against_golden(tb, golden, d)


@pytest.mark.gpu
def test_press_dataset_batch_size_does_not_change_results(golden, tmp_path):
    """One simulation at a time (the reference's per-thread job) and all four
    stepped together give the same dataset."""
    tb = _tb()
    for batch in (1, 3):
        d = str(tmp_path / f"b{batch}")
        assert tb.dataset.run_press_dataset(HARNESS, d, batch=batch) == (12, 0)
        _check_against_golden(tb, golden, d)


@pytest.mark.gpu
def test_press_dataset_resume(golden, tmp_path):
    """Complete (object, position) groups are kept and skipped; incomplete
    ones are re-run (harness.cpp:165-178)."""
    tb = _tb()
    d = str(tmp_path / "ds")
    assert tb.dataset.run_press_dataset(HARNESS, d) == (12, 0)
    assert tb.dataset.run_press_dataset(HARNESS, d) == (12, 4)
    man = os.path.join(d, "manifest.csv")
    with open(man) as f:
        lines = f.read().splitlines()
    # drop one depth row of dots/p1 and delete its image: that group re-runs
    dropped = [l for l in lines if l.startswith("dots,1,")][1]
    os.remove(os.path.join(d, dropped.split(",")[8]))
    with open(man, "w") as f:
        f.write("\n".join(l for l in lines if l != dropped) + "\n")
    assert tb.dataset.run_press_dataset(HARNESS, d) == (12, 3)
    _check_against_golden(tb, golden, d)


@pytest.mark.gpu
def test_image_metrics_match_reference(golden):
    tb = _tb()
    pairs = golden["metric_pairs"]
    a = np.array([golden[str(x)] for x, _ in pairs])
    b = np.array([golden[str(y)] for _, y in pairs])
    m = tb.metrics.compare_batch(a, b)
    ref = golden["metrics"]
    np.testing.assert_allclose(m[:, 0], ref[:, 0], rtol=0, atol=1e-10)
    np.testing.assert_array_equal(m[:, 1:], ref[:, 1:])  # psnr, mae exact (inf included)
    nm = tb.metrics.compare(golden["noise_a"], golden["noise_b"])
    assert nm[0] == pytest.approx(float(golden["noise_metrics"][0]), abs=1e-10)
    assert nm[1:] == tuple(golden["noise_metrics"][1:])
    with pytest.raises(tb.ShapeMismatch):
        tb.metrics.compare(np.zeros((7, 9, 3), np.uint8), np.zeros((7, 9, 3), np.uint8))


@pytest.mark.gpu
def test_image_metrics_exact_on_random_pairs():
    """PSNR and MAE bit-equal to the reference's metrics::compare on random
    noise pairs (the device sums squared / absolute differences in integers;
    PSNR's log10 is taken on the host, the reference's own call — the device
    log10 differed in the last ulp on some pairs), SSIM to 1e-12."""
    from oracle import refpy  # the reference, as the checker

    tb = _tb()
    rng = np.random.default_rng(11)
    a = rng.integers(0, 256, (16, 48, 64, 3), dtype=np.uint8)
    b = np.clip(a.astype(np.int32) + rng.integers(-20, 21, a.shape), 0, 255).astype(np.uint8)
    m = tb.metrics.compare_batch(a, b)
    for i in range(len(a)):
        r = refpy.image_metrics(a[i], b[i])
        assert abs(m[i, 0] - r[0]) <= 1e-12
        assert (m[i, 1], m[i, 2]) == (r[1], r[2])


@pytest.mark.gpu
def test_compare_datasets(tmp_path):
    """compare_datasets over two harness outputs: identical -> SSIM 1, PSNR
    inf, MAE 0; a perturbed copy -> per-pair metrics equal metrics.compare."""
    tb = _tb()
    a = str(tmp_path / "a")
    tb.dataset.run_press_dataset(HARNESS, a)
    b = str(tmp_path / "b")
    shutil.copytree(a, b)
    agg = tb.dataset.compare_datasets(a, b, str(tmp_path / "same.csv"))
    assert agg["pairs"] == 12 and agg["ssim_mean"] == 1.0 and agg["mae_mean"] == 0.0
    assert agg["psnr_mean"] == float("inf")
    rng = np.random.default_rng(3)
    with open(os.path.join(a, "manifest.csv")) as f:
        imgs = [l.split(",")[8] for l in f.read().splitlines()[1:]]
    for rel in imgs:
        img = tb.load_png(os.path.join(b, rel)).astype(int)
        img = np.clip(img + rng.integers(-6, 7, img.shape), 0, 255).astype(np.uint8)
        tb.save_png(img, os.path.join(b, rel))
    csv = str(tmp_path / "diff.csv")
    agg = tb.dataset.compare_datasets(a, b, csv)
    per = np.array([tb.metrics.compare(tb.load_png(os.path.join(a, r)),
                                       tb.load_png(os.path.join(b, r))) for r in sorted(imgs)])
    assert agg["pairs"] == 12
    assert agg["ssim_mean"] == pytest.approx(per[:, 0].mean(), rel=1e-12)
    assert agg["psnr_mean"] == pytest.approx(per[:, 1].mean(), rel=1e-12)
    assert agg["mae_std"] == pytest.approx(per[:, 2].std(ddof=1), rel=1e-9)
    with open(csv) as f:
        lines = f.read().splitlines()
    assert lines[0] == "object,position_index,depth_index,ssim,psnr_db,mae_pct"
    assert len(lines) == 1 + 12 + 2 and lines[-2].startswith("mean,,,")
