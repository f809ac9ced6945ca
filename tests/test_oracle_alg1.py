"""Pins of the oracle's NEXT-2 histogram voting, Alg. 1 (
DESIGN.md R22), on hand-derived cases: a fronto-parallel plane seen along the
optical axis, where a = depth - Z is known for every voxel."""
import json
import os

import numpy as np

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def axis_camera(f, w=64, h=64, weight=1):
    return {"origin": (0.0, 0.0, 0.0), "rot": np.eye(3), "fx": f, "fy": f, "cx": w / 2 + 0.5, "cy": h / 2 + 0.5,
            "width": w, "height": h, "vote_weight": weight}


def axis_counts(cam, depth, zs):
    """One voxel column on the optical axis at camera-frame depths zs (voxel size 1)."""
    c = oracle.alg1_vote([cam], [depth], 1, 1, 0, len(zs), origin=(0.0, 0.0, float(zs[0])))
    return c[:, 0, 0, :]


def test_plane_bins_golden():
    g = json.load(open(os.path.join(GOLD, "alg1_plane.json")))
    cam = axis_camera(g["f"])
    depth = np.full((64, 64), g["plane_depth"], np.float32)
    zs = list(range(g["z_first"], g["z_last"] + 1))
    c = axis_counts(cam, depth, zs)
    for z, want in zip(zs, g["bin_by_z"]):
        row = c[z - zs[0]]
        if want is None:
            assert row.sum() == 0, z
        else:
            assert row.sum() == 1 and row[want] == 1, (z, row)


def test_vote_weight_and_additivity():
    depth = np.full((64, 64), 50.0, np.float32)
    zs = list(range(40, 65))
    one = axis_counts(axis_camera(100.0), depth, zs)
    five = axis_counts(axis_camera(100.0, weight=5), depth, zs)
    assert np.array_equal(five, 5 * one)
    two = oracle.alg1_vote([axis_camera(100.0)] * 2, [depth] * 2, 1, 1, 0, 25, origin=(0.0, 0.0, 40.0))
    assert np.array_equal(two[:, 0, 0], 2 * one)


def test_mipmap_level_selection():
    # pixel checkerboard 40 / 60: level 0 reads 40 or 60, level 1 reads the 2x2 mean 50.
    yy, xx = np.mgrid[0:64, 0:64]
    depth = np.where((xx + yy) % 2 == 0, 40.0, 60.0).astype(np.float32)
    z = [50]
    # f = 100: projected diameter 2 r f / Z = 2 >= sqrt(2) -> level 1 -> depth 50 -> a = 0 -> bin 4
    c1 = axis_counts(axis_camera(100.0), depth, z)[0]
    assert c1[4] == 1
    # f = 60: diameter 1.2 < sqrt(2) -> level 0 -> the axis pixel (32, 32): (32+32) even -> 40 -> a = -10 < -9 -> no vote
    c0 = axis_counts(axis_camera(60.0), depth, z)[0]
    assert c0.sum() == 0


def test_behind_and_outside():
    depth = np.full((64, 64), 50.0, np.float32)
    cam = axis_camera(100.0)
    behind = oracle.alg1_vote([cam], [depth], 1, 1, 0, 3, origin=(0.0, 0.0, -5.0))
    assert behind.sum() == 0
    outside = oracle.alg1_vote([cam], [depth], 1, 1, 0, 1, origin=(500.0, 0.0, 50.0))
    assert outside.sum() == 0
    nan = np.full((64, 64), np.nan, np.float32)
    assert oracle.alg1_vote([cam], [nan], 1, 1, 0, 1, origin=(0.0, 0.0, 50.0)).sum() == 0
