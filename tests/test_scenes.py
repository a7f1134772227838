"""Seeded input generators (scenes/) are deterministic and shaped as DESIGN.md states."""
import numpy as np

from scenes import scene_c1, scene_c2, advance_scene


def test_c1_shape():
    sc = scene_c1()
    assert (sc.W, sc.H) == (64, 64) and int(sc.static.sum()) == 208 and sc.n_tracks == 0


def test_c2_deterministic_and_shaped():
    a, b = scene_c2(4), scene_c2(4)
    assert np.array_equal(a.static, b.static) and np.array_equal(a.tracks, b.tracks)
    assert a.n_tracks == 20 and a.static.shape == (512, 512)
    assert a.static[a.goal[1], a.goal[0]] == 0
    rx, ry = int(a.robot[0] / 0.1), int(a.robot[1] / 0.1)
    assert a.static[ry, rx] == 0
    c = scene_c2(5)
    assert not np.array_equal(a.tracks, c.tracks)


def test_advance_scene_moves_robot_and_obstacles():
    a = scene_c2(0)
    b = advance_scene(a, 10)
    assert b.robot[0] > a.robot[0] and b.robot[1] > a.robot[1]
    assert np.array_equal(advance_scene(a, 10).tracks, b.tracks)
    assert not np.allclose(b.truth[:, :2], a.truth[:, :2])
