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
