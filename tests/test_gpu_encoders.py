"""Output encoders on the device (codecs.cu) against the C restatement of
proj/src/io.cpp's rasters (oracle/ps_oracle.c, pinned to the reference's own
known answers in tests/test_oracle.py): KITTI 16-bit, PFM, point cloud —
on hand-made maps, on pipeline outputs, and on a resident batch."""
import numpy as np
import pytest

import paper_1511_00758_b200 as ps

pytestmark = pytest.mark.gpu


def random_map(rng, h, w, lo=0.0, hi=127.0, p_valid=0.7):
    d = rng.uniform(lo, hi, (h, w)).astype(np.float32)
    ok = (rng.random((h, w)) < p_valid).astype(np.uint8)
    return d, ok


def test_kitti_and_pfm_equal_oracle(ctx, orc):
    rng = np.random.default_rng(7)
    for h, w in [(16, 20), (37, 53), (120, 160)]:
        d, ok = random_map(rng, h, w)
        d[0, 0], ok[0, 0] = 0.0, 1          # clamps to raw 1
        d[0, 1], ok[0, 1] = 1000.0, 1       # clamps to 65535
        d[0, 2], ok[0, 2] = 0.5 / 256, 1    # raw 0.5 rounds away from zero -> 1
        d[0, 3], ok[0, 3] = 2.5 / 256, 1    # raw 2.5 -> 3
        d[0, 4], ok[0, 4] = -0.0, 1         # not negative: raw 1
        want, neg = orc.encode_kitti16(d, ok)
        assert neg == -1
        assert np.array_equal(ctx.encode_kitti16(d, ok), want)
        assert np.array_equal(ctx.encode_pfm(d, ok).view(np.uint32), orc.encode_pfm(d, ok).view(np.uint32))
    # batched form: frames stacked
    d, ok = random_map(rng, 3 * 40, 64)
    d, ok = d.reshape(3, 40, 64), ok.reshape(3, 40, 64)
    k = ctx.encode_kitti16(d, ok)
    p = ctx.encode_pfm(d, ok)
    for f in range(3):
        assert np.array_equal(k[f], orc.encode_kitti16(d[f], ok[f])[0])
        assert np.array_equal(p[f], orc.encode_pfm(d[f], ok[f]))


def test_kitti_negative_disparity_is_an_error(ctx):
    d = np.zeros((16, 16), np.float32)
    ok = np.zeros((16, 16), np.uint8)
    d[3, 3], ok[3, 3] = -1.0, 1
    d[9, 1], ok[9, 1] = -7.0, 1
    with pytest.raises(ps.NegativeDisparity, match="-1.000000"):  # the first, row-major
        ctx.encode_kitti16(d, ok)
    ok[3, 3] = 0  # an invalid pixel's value is never looked at
    with pytest.raises(ps.NegativeDisparity, match="-7.000000"):
        ctx.encode_kitti16(d, ok)


def test_point_cloud_equals_oracle(ctx, orc):
    rng = np.random.default_rng(8)
    d, ok = random_map(rng, 90, 120, lo=0.0, hi=40.0)
    img = rng.integers(0, 256, (90, 120), dtype=np.uint8)
    for calib, lo in [((700.0, 0.54, 60.0, 45.0), 0.5), ((100.0, 0.25, 0.0, 0.0), 0.0),
                      ((718.856, 0.5371657, 607.1928, 185.2157), 3.0)]:
        xyz, inten = ctx.point_cloud(d, ok, img, calib, lo)
        oxyz, ointen = orc.point_cloud(d, ok, img, calib, lo)
        assert np.array_equal(xyz.view(np.uint32), oxyz.view(np.uint32))
        assert np.array_equal(inten, ointen)
    with pytest.raises(ps.EmptyCloud):
        ctx.point_cloud(d, np.zeros_like(ok), img, (100.0, 0.5, 0.0, 0.0))
    with pytest.raises(ps.InvalidConfig):
        ctx.point_cloud(d, ok, img, (100.0, 0.0, 0.0, 0.0))


def test_resident_downloads_equal_host_encoding(ctx, orc):
    """ps_download_* encode the last run's maps on the device; equal to encoding
    the downloaded maps on the host, and a failed frame encodes as all-invalid."""
    c = ps.BASELINE_CONFIGS[2]
    cfg = ps.baseline_config(2)
    n = 4
    L, R = ps.synth_batch(n, c["width"], c["height"], c["n_planes"], c["max_disparity"],
                          c["ground"], c["sigma"], seed=90)
    L[2] = 128
    R[2] = 128
    res = ctx.run_batch(L, R, cfg, unchecked_cell=True, raise_on_failure=False)
    assert list(res["status"]) == [0, 0, 7, 0]
    for which, dk, vk in [(0, "disparity", "disparity_valid"), (1, "dense", "dense_valid")]:
        k = ctx.download_kitti16(which)
        p = ctx.download_pfm(which)
        for f in range(n):
            assert np.array_equal(k[f], orc.encode_kitti16(res[dk][f], res[vk][f])[0]), (which, f)
            assert np.array_equal(p[f], orc.encode_pfm(res[dk][f], res[vk][f])), (which, f)
        assert (k[2] == 0).all() and (p[2] == -1.0).all()
    calib = (718.856, 0.5371657, 319.5, 239.5)
    xyz, inten = ctx.download_point_cloud(1, calib)
    oxyz, ointen = orc.point_cloud(res["disparity"][1], res["disparity_valid"][1], L[1], calib)
    assert len(xyz) > 1000
    assert np.array_equal(xyz.view(np.uint32), oxyz.view(np.uint32)) and np.array_equal(inten, ointen)
    with pytest.raises(ps.EmptyCloud):
        ctx.download_point_cloud(2, calib)
