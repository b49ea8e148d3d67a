"""CLI host logic (no GPU): option precedence, config files, validation and
exit codes of the reference CLI (src/cli.py:1-16, 124-165, 395-425)."""
import os

import pytest

from paper_1901_03088_b200 import cli


def _args(argv):
    return cli.build_parser().parse_args(argv)


def test_defaults_and_precedence(tmp_path, monkeypatch):
    conf = tmp_path / "c.conf"
    conf.write_text("# comment\nlambda = 0.2\nseed = 5\nworkers = 3\nverbose = yes\n")
    monkeypatch.setenv(cli.WORKERS_ENV, "7")
    cfg = cli.resolve(_args(["fit", "x.png", "--out", "p.txt"]))
    assert cfg["lam"] == 0.1 and cfg["workers"] == 7 and cfg["precision"] == "exact"
    cfg = cli.resolve(_args(["fit", "x.png", "--out", "p", "--config", str(conf)]))
    assert (cfg["lam"], cfg["seed"], cfg["workers"], cfg["verbose"]) == (0.2, 5, 3, True)
    cfg = cli.resolve(_args(["fit", "x.png", "--out", "p", "--config", str(conf), "--seed", "9",
                             "--workers", "1"]))
    assert (cfg["seed"], cfg["workers"]) == (9, 1)


@pytest.mark.parametrize("argv", [
    ["fit", "x.png", "--out", "p", "--white-threshold", "255"],
    ["fit", "x.png", "--out", "p", "--background-cutoff", "0"],
    ["fit", "x.png", "--out", "p", "--rel-tol", "0"],
    ["fit", "x.png", "--out", "p", "--patch-size", "0"],
    ["fit", "x.png", "--out", "p", "--precision", "approximate"],
    ["fit", "x.png", "--out", "p", "--lambda", "-1"],
])
def test_invalid_options_exit_2(argv):
    assert cli.main(argv) == cli.EXIT_INPUT


def test_config_errors_exit_2(tmp_path):
    bad = tmp_path / "bad.conf"
    bad.write_text("no equals sign here\n")
    assert cli.main(["fit", "x.png", "--out", "p", "--config", str(bad)]) == 2
    bad.write_text("unknown-option = 1\n")
    assert cli.main(["fit", "x.png", "--out", "p", "--config", str(bad)]) == 2
    bad.write_text("verbose = maybe\n")
    assert cli.main(["fit", "x.png", "--out", "p", "--config", str(bad)]) == 2


def test_input_errors_exit_2_before_any_gpu_work(tmp_path, monkeypatch):
    assert cli.main(["fit", str(tmp_path / "missing.png"), "--out", "p"]) == 2
    txt = tmp_path / "notes.png"
    txt.write_text("not an image")
    assert cli.main(["fit", str(txt), "--out", "p"]) == 2
    assert cli.main(["batch", str(tmp_path / "nodir"), "--profile", "p", "--out", "o"]) == 2
    empty = tmp_path / "empty"
    empty.mkdir()
    assert cli.main(["batch", str(empty), "--profile", "p", "--out", "o"]) == 2
    monkeypatch.setenv(cli.WORKERS_ENV, "many")
    assert cli.main(["fit", "x.png", "--out", "p"]) == 2
    assert cli.main(["bench", "12,abc"]) == 2
    assert cli.main([]) == 2                          # argparse usage error


def test_exit_code_mapping():
    E = cli.E
    assert cli.exit_code_of(E.BlankSlideError("x")) == 3
    assert cli.exit_code_of(E.InsufficientPixelsError("x")) == 3
    assert cli.exit_code_of(E.StainAbsentError("x")) == 4
    assert cli.exit_code_of(E.DegenerateStainError("x")) == 4
    assert cli.exit_code_of(E.ProfileError("x")) == 2
    assert cli.exit_code_of(E.UnsupportedFormatError("x")) == 2
    assert cli.exit_code_of(cli.OutputError("x")) == 5
    assert cli.exit_code_of(FileNotFoundError("x")) == 2


def test_file_io_roundtrip(tmp_path):
    import numpy as np

    from paper_1901_03088_b200 import image_io as io

    a = (np.arange(20 * 30 * 3) % 251).astype(np.uint8).reshape(20, 30, 3)
    for ext in ("png", "npy"):
        path = tmp_path / f"a.{ext}"
        with io.open_writer(path, 30, 20) as w:
            w.write_strip(io.PixelBlock(0, 0, a[:7]))
            w.write_strip(io.PixelBlock(0, 7, a[7:]))
        with io.open_slide(path) as s:
            assert np.array_equal(s.read_region(0, 0, 30, 20).pixels, a)
    with pytest.raises(ValueError):               # incomplete image leaves no file
        with io.open_writer(tmp_path / "b.png", 30, 20) as w:
            w.write_strip(io.PixelBlock(0, 0, a[:7]))
    assert not os.path.exists(tmp_path / "b.png")
    with pytest.raises(cli.E.UnsupportedFormatError):
        io.open_writer(tmp_path / "c.jpg", 30, 20)


@pytest.mark.parametrize("comp,big", [("deflate", False), ("none", False), ("deflate", True)])
def test_tiff_codec_roundtrip_and_pillow(tmp_path, comp, big):
    import numpy as np
    from PIL import Image

    from paper_1901_03088_b200 import image_io as io
    from paper_1901_03088_b200 import tiff

    rng = np.random.default_rng(1)
    a = rng.integers(0, 256, size=(600, 530, 3), dtype=np.uint8)
    p = tmp_path / "t.tif"
    w = tiff.TiffTileWriter(p, 530, 600, compression=comp, bigtiff=big)
    for y in range(0, 600, 250):
        w.write(a[y:y + 250])
    w.close()
    with io.open_slide(p) as s:
        assert (s.width, s.height) == (530, 600)
        assert np.array_equal(s.read_region(0, 0, 530, 600).pixels, a)
        assert np.array_equal(s.read_region(97, 255, 300, 211).pixels, a[255:466, 97:397])
    if not big:                                   # libtiff (through Pillow) reads ours
        with Image.open(p) as im:
            assert np.array_equal(np.asarray(im.convert("RGB")), a)


def test_tiff_reads_pillow_strips_and_rejects_unsupported(tmp_path):
    import numpy as np
    from PIL import Image

    from paper_1901_03088_b200 import image_io as io

    a = np.random.default_rng(2).integers(0, 256, size=(300, 200, 3), dtype=np.uint8)
    for comp in ("raw", "tiff_adobe_deflate"):
        p = tmp_path / f"{comp}.tif"
        Image.fromarray(a).save(p, compression=comp)
        with io.open_slide(p) as s:
            assert np.array_equal(s.read_region(0, 0, 200, 300).pixels, a)
    p = tmp_path / "lzw.tif"
    Image.fromarray(a).save(p, compression="tiff_lzw")
    with pytest.raises(cli.E.UnsupportedFormatError):
        io.open_slide(p)
    p = tmp_path / "gray.tif"
    Image.fromarray(a[..., 0]).save(p)
    with pytest.raises(cli.E.UnsupportedFormatError):
        io.open_slide(p)
    good = tmp_path / "raw.tif"
    bad = tmp_path / "cut.tif"
    bad.write_bytes(good.read_bytes()[:5000])
    with pytest.raises(cli.E.CorruptImageError):
        io.open_slide(bad)


def test_tiff_strip_writer_through_open_writer(tmp_path):
    import numpy as np

    from paper_1901_03088_b200 import image_io as io

    a = np.random.default_rng(3).integers(0, 256, size=(513, 300, 3), dtype=np.uint8)
    with io.open_writer(tmp_path / "o.tiff", 300, 513) as w:
        for y in range(0, 513, 100):
            w.write_strip(io.PixelBlock(0, y, a[y:y + 100]))
    with io.open_slide(tmp_path / "o.tiff") as s:
        assert np.array_equal(s.read_region(0, 0, 300, 513).pixels, a)
    with pytest.raises(ValueError):
        with io.open_writer(tmp_path / "p.tif", 300, 513) as w:
            w.write_strip(io.PixelBlock(0, 0, a[:100]))
    assert not os.path.exists(tmp_path / "p.tif")


def test_png_strip_writer_streams_with_bounded_memory(tmp_path):
    """The PNG sink encodes strip by strip (src/image_io.py:316-358): the
    file exists once opened, holds IDAT data before close, decodes to the
    written pixels, and an unwritable path fails on open."""
    import numpy as np
    from PIL import Image

    from paper_1901_03088_b200 import image_io as io

    rng = np.random.default_rng(4)
    img = rng.integers(0, 256, size=(300, 257, 3), dtype=np.uint8)
    path = tmp_path / "s.png"
    w = io.open_writer(path, 257, 300)
    assert isinstance(w, io.PngStripWriter) and os.path.exists(path)
    for y in range(0, 300, 64):
        w.write_strip(io.PixelBlock(0, y, img[y:y + 64]))
        if y >= 128:
            assert os.path.getsize(path) > 1000          # data already on disk
    w.close()
    assert np.array_equal(np.asarray(Image.open(path)), img)
    with pytest.raises(OSError):
        io.open_writer(tmp_path / "missing" / "x.png", 10, 10)


def test_png_bytes_equal_the_reference_writer(tmp_path):
    """A PNG written strip by strip is byte-identical to the one the
    reference's own PngStripWriter wrote (tests/golden/png_ref_strips.png,
    oracle/make_golden.py --png), and reads back to the same pixels."""
    import numpy as np

    from paper_1901_03088_b200 import image_io as io

    golden = os.path.join(os.path.dirname(__file__), "golden", "png_ref_strips.png")
    h, w = 37, 53
    px = np.random.default_rng(2024).integers(0, 256, size=(h, w, 3), dtype=np.uint8)
    path = tmp_path / "ours.png"
    with io.open_writer(path, w, h) as wr:
        for y in range(0, h, 10):
            wr.write_strip(io.PixelBlock(0, y, px[y:y + 10]))
    assert open(path, "rb").read() == open(golden, "rb").read()
    src = io.open_slide(golden)                 # our reader on the reference's file
    assert np.array_equal(np.asarray(src.read_region(0, 0, w, h).pixels), px)
