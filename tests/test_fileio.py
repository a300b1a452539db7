"""File formats vs files written by the reference's fileio (tests/golden/fileio/)."""

import dataclasses
import json
import shutil

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2603_28756_b200 import fileio
from paper_2603_28756_b200.geometry import ImageGrid, Sinogram, Volume
from paper_2603_28756_b200.solver import IterationRecord

G = GOLDEN / "fileio"


def test_round_trip_is_byte_identical(tmp_path):
    for name, kind in (("vol.raw", Volume), ("img.raw", ImageGrid), ("sino.raw", Sinogram)):
        obj = fileio.load_array(G / name)
        assert isinstance(obj, kind)
        out = fileio.save_array(tmp_path / name, obj)
        assert out.read_bytes() == (G / name).read_bytes()
        assert json.loads((tmp_path / (name + ".json")).read_text()) == \
            json.loads((G / (name + ".json")).read_text())
    vol = fileio.load_array(G / "vol.raw")
    assert vol.pixel_size == 0.5 and vol.data.shape == (3, 5, 5)
    sino = fileio.load_array(G / "sino.raw")
    np.testing.assert_array_equal(sino.angles, np.linspace(0, np.pi, 6, endpoint=False))


def test_corrupt_files_rejected(tmp_path):
    shutil.copy(G / "vol.raw", tmp_path / "v.raw")
    shutil.copy(G / "vol.raw.json", tmp_path / "v.raw.json")
    (tmp_path / "v.raw").write_bytes((G / "vol.raw").read_bytes()[:-8])
    with pytest.raises(ValueError, match="payload"):
        fileio.load_array(tmp_path / "v.raw")
    head = json.loads((G / "vol.raw.json").read_text())
    head["dtype"] = "<f4"
    (tmp_path / "v.raw").write_bytes((G / "vol.raw").read_bytes())
    (tmp_path / "v.raw.json").write_text(json.dumps(head))
    with pytest.raises(ValueError, match="dtype"):
        fileio.load_array(tmp_path / "v.raw")
    with pytest.raises(TypeError):
        fileio.save_array(tmp_path / "x.raw", np.zeros(3))


def test_plan_parse_matches_reference():
    plan = fileio.load_plan(G / "plan.toml")
    want = json.loads((G / "plan_parsed.json").read_text())
    got = dataclasses.asdict(plan)
    got["init_volume"] = plan.init_volume.name
    got["iters_per_level"] = list(got["iters_per_level"])
    assert json.loads(json.dumps(got, default=str)) == want
    assert plan.resolve_params(0.2).sigma == 0.2


@pytest.mark.parametrize("text,match", [
    ("[geometry]\nimage_side = 8\n[bogus]\nx = 1\n", "unknown plan section"),
    ("[geometry]\nimage_side = 8\nfoo = 1\n", "unknown keys"),
    ("[qggmrf]\nsigma = 1.0\n", "image_side"),
    ("[geometry]\nimage_side = 8\n[qggmrf]\nsigma = \"big\"\n", "sigma"),
    ("[geometry]\nimage_side = 8\n[solver]\nlipschitz = \"x\"\n", "lipschitz"),
    ("[geometry]\nimage_side = 8\n[files]\ninit_volume = \"missing.raw\"\n", "does not exist"),
])
def test_plan_schema_errors(tmp_path, text, match):
    (tmp_path / "p.toml").write_text(text)
    with pytest.raises(ValueError, match=match):
        fileio.load_plan(tmp_path / "p.toml")


def test_convergence_csv_matches_reference(tmp_path):
    recs = [IterationRecord(i, 100.0 / (i + 1), 90.0 / (i + 1), 1.0 / 3, 0.5 ** i, 0.01 * i,
                            i == 2) for i in range(4)]
    out = fileio.write_convergence_csv(tmp_path / "c.csv", [(r, i % 2, 1) for i, r in enumerate(recs)],
                                       {"seed": 7, "image_side": 64, "init": "fbp"})
    assert out.read_text() == (G / "conv.csv").read_text()


def test_export_slice_matches_reference(tmp_path):
    img = ImageGrid(np.outer(np.arange(6.0), np.ones(6)))
    out = fileio.export_slice(tmp_path / "prev.pgm", img)
    assert out.name == "prev_w0_5.pgm"
    assert out.read_bytes() == (G / "prev_w0_5.pgm").read_bytes()
    with pytest.raises(ValueError):
        fileio.export_slice(tmp_path / "x.jpg", img)
