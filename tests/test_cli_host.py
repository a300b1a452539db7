"""CLI host-side behaviour (no GPU): phantom files, argument errors, exit codes."""

import numpy as np

from paper_2603_28756_b200 import cli, fileio
from paper_2603_28756_b200.phantoms import shepp_logan


def test_phantom_command_writes_reference_format(tmp_path):
    out = tmp_path / "p.raw"
    assert cli.main(["phantom", "--kind", "shepp-logan", "--side", "32", "--slices", "3",
                     "--out", str(out)]) == cli.EXIT_OK
    vol = fileio.load_array(out)
    np.testing.assert_array_equal(vol.data, shepp_logan(32, True, 3).data)
    assert cli.main(["phantom", "--kind", "disk", "--side", "16", "--out",
                     str(tmp_path / "d.raw")]) == cli.EXIT_OK


def test_exit_codes(tmp_path, monkeypatch):
    assert cli.main(["phantom", "--kind", "cube", "--side", "8", "--out", "x"]) == 2
    assert cli.main(["mbir", "--sino", str(tmp_path / "none.raw"), "--plan",
                     str(tmp_path / "none.toml"), "--out", str(tmp_path / "r.raw")]) == cli.EXIT_IO
    (tmp_path / "bad.toml").write_text("[geometry]\nimage_side = 8\n[nope]\n")
    assert cli.main(["mbir", "--sino", "s", "--plan", str(tmp_path / "bad.toml"),
                     "--out", "r"]) == cli.EXIT_USAGE
    monkeypatch.setenv("TOMOFORGE_THREADS", "2")
    assert cli._cap_workers(8) == 2
    monkeypatch.setenv("TOMOFORGE_THREADS", "many")
    assert cli.main(["phantom", "--kind", "disk", "--side", "8", "--radius", "9",
                     "--out", str(tmp_path / "d.raw")]) == cli.EXIT_USAGE


def test_bench_options_match_reference():
    """`bench` takes the reference's categories and options (cli.py:223-233)."""
    from paper_2603_28756_b200 import cli

    ap = cli.build_parser()
    for cat in ("toeplitz", "init", "multires", "scaling"):
        a = ap.parse_args(["bench", cat, "--out", "x.csv"])
        assert a.category == cat and a.sizes == [32, 64, 128, 256] and a.side == 256
        assert a.slices == 32 and a.angles == 60 and a.iters == 3 and a.workers == [1, 2, 4]
