""".capt dumps written by the REFERENCE's save_capt (tree.py:276-288;
fixtures from tests/golden/make_golden.py): load_capt reads them straight
into the device layout, save_capt writes them back byte for byte, and the
loaded trees answer the reference's own masks (computed by the reference on
its load_capt of the same file)."""

import os

import numpy as np
import pytest

from conftest import GOLDEN, load_golden

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2406_02807_b200")


@pytest.mark.parametrize("name", ["ref3d", "ref2d"])
def test_reference_written_capt_round_trip(name, tmp_path):
    path = os.path.join(GOLDEN, f"{name}.capt")
    tree = P.load_capt(path)
    # r_min / r_max come back as their fp32 values, as in the reference (tree.py:297,318)
    assert tree.r_min == float(np.float32(tree.r_min))
    out = tmp_path / "back.capt"
    P.save_capt(tree, out)
    assert open(path, "rb").read() == open(out, "rb").read()
    z = load_golden("capt_files.npz")
    c, r = z[f"{name}/centers"], z[f"{name}/radii"]
    exp = np.unpackbits(z[f"{name}/mask"])[: len(r)].astype(bool)
    assert np.array_equal(P.collides_many(tree, c, r), exp)


def test_reference_written_capt_rejects_corruption(tmp_path):
    raw = open(os.path.join(GOLDEN, "ref3d.capt"), "rb").read()
    bad = tmp_path / "t.capt"
    bad.write_bytes(raw[:-4])
    with pytest.raises(ValueError):
        P.load_capt(bad)
    bad.write_bytes(raw + b"\0")
    with pytest.raises(ValueError, match="trailing"):
        P.load_capt(bad)
    bad.write_bytes(b"NOTCAPT!" + raw[8:])
    with pytest.raises(ValueError, match="magic"):
        P.load_capt(bad)
