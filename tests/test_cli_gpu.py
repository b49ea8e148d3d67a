"""CLI end to end on the GPU: fit → profile, normalize (--target / --profile),
batch with per-file failures, bench CSV — outputs byte-identical to the
reference algorithm (oracle) on the same PNG inputs."""
import os

import numpy as np
import pytest

from oracle import spcn_oracle as orc

pytestmark = pytest.mark.gpu


def _png(path, px):
    from PIL import Image

    Image.fromarray(px, mode="RGB").save(path)


def _read(path):
    from PIL import Image

    with Image.open(path) as im:
        return np.asarray(im.convert("RGB"))


def test_cli_fit_normalize_batch(tmp_path, capsys):
    from paper_1901_03088_b200 import cli

    src, _, _ = orc.render(420, 300, 1, i0=(250, 244, 252), tissue_fraction=0.6)
    tgt, _, _ = orc.render(380, 260, 2, tissue_fraction=0.5)
    _png(tmp_path / "src.png", src)
    _png(tmp_path / "tgt.png", tgt)
    fs, ft = orc.fit_params(src), orc.fit_params(tgt)
    ref = orc.run_transform(src, fs, ft, workers=1)

    prof = tmp_path / "tgt.profile"
    assert cli.main(["fit", str(tmp_path / "tgt.png"), "--out", str(prof)]) == 0
    assert capsys.readouterr().out.strip() == str(prof)
    out = tmp_path / "out.png"
    assert cli.main(["normalize", str(tmp_path / "src.png"), "--target",
                     str(tmp_path / "tgt.png"), "--out", str(out),
                     "--stats-csv", str(tmp_path / "s.csv")]) == 0
    assert np.array_equal(_read(out), ref)
    assert (tmp_path / "s.csv").read_text().count("\n") >= 2
    from paper_1901_03088_b200 import tiff

    tw = tiff.TiffTileWriter(tmp_path / "src.tif", src.shape[1], src.shape[0])
    tw.write(src)
    tw.close()
    out_t = tmp_path / "out.tif"
    assert cli.main(["normalize", str(tmp_path / "src.tif"), "--target",
                     str(tmp_path / "tgt.png"), "--out", str(out_t)]) == 0
    from paper_1901_03088_b200 import image_io

    with image_io.open_slide(out_t) as s:
        assert np.array_equal(s.read_region(0, 0, s.width, s.height).pixels, ref)
    out2 = tmp_path / "out2.npy"
    assert cli.main(["normalize", str(tmp_path / "src.png"), "--profile", str(prof),
                     "--out", str(out2)]) == 0
    assert np.array_equal(np.load(out2), ref)

    d = tmp_path / "in"
    d.mkdir()
    _png(d / "a.png", src)
    _png(d / "b.png", np.full((64, 64, 3), 255, np.uint8))      # blank: fails, batch goes on
    np.save(d / "c.npy", src)
    capsys.readouterr()
    rc = cli.main(["batch", str(d), "--profile", str(prof), "--out", str(tmp_path / "o")])
    assert rc == cli.EXIT_BATCH_FAILURES
    cap = capsys.readouterr()
    assert "b.png" in cap.err and cap.out.split() == [str(tmp_path / "o" / "a.png"),
                                                     str(tmp_path / "o" / "c.npy")]
    assert np.array_equal(_read(tmp_path / "o" / "a.png"), ref)
    assert np.array_equal(np.load(tmp_path / "o" / "c.npy"), ref)
    assert not os.path.exists(tmp_path / "o" / "b.png")


def test_cli_exit_codes_blank_and_bench(tmp_path, capsys):
    from paper_1901_03088_b200 import cli

    _png(tmp_path / "white.png", np.full((80, 80, 3), 255, np.uint8))
    assert cli.main(["fit", str(tmp_path / "white.png"), "--out", str(tmp_path / "p")]) == 3
    capsys.readouterr()
    assert cli.main(["bench", "128,256"]) == 0
    lines = capsys.readouterr().out.strip().splitlines()
    assert lines[0] == "size,stage,seconds,pixels,patches" and len(lines) > 3
