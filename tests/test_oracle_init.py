"""CPU: pin the init_from_depth restatement (oracle/psplat_oracle.c) to the
reference's scene_init.cpp compiled from its own sources, bit for bit."""
import numpy as np
import pytest

from oracle.oracle import Camera, RefScenes


def _same(a, b):
    assert a.n == b.n
    for x, y in [(a.center, b.center), (a.rotation, b.rotation), (a.radii, b.radii), (a.ids, b.ids)]:
        assert np.array_equal(x, y)


@pytest.fixture(scope="module")
def room(ref):
    rs = RefScenes()
    spec = (4.0, 4.0, 3.0, 1, 7)
    cams = list(rs.room_views(*spec, 40, 7, 48, 36))[:12]
    td, tn = rs.render_ground_truth(spec, (Camera * len(cams))(*cams))
    return cams, td, tn


@pytest.mark.parametrize("n,seed,scale", [(64, 7, 0.5), (500, 1, 0.5), (3000, 2, 0.25)])
def test_init_from_depth_bitwise_vs_reference(ref, orc, room, n, seed, scale):
    cams, td, tn = room
    _same(ref.init_from_depth(cams, td, tn, n, seed, scale), orc.init_from_depth(cams, td, tn, n, seed, scale))


def test_init_from_depth_edge_cases(ref, orc, room):
    cams, td, tn = room
    # one primitive: fallback radius from the bounds; more primitives than pixels
    _same(ref.init_from_depth(cams[:1], td, tn, 1, 3), orc.init_from_depth(cams[:1], td, tn, 1, 3))
    npx = cams[0].width * cams[0].height
    big = ref.init_from_depth(cams[:1], td[:npx], tn[:3 * npx], npx + 10, 3)
    _same(big, orc.init_from_depth(cams[:1], td[:npx], tn[:3 * npx], npx + 10, 3))
    assert big.n <= npx
    # errors: n < 1 (invalid_argument), no valid pixel (runtime_error)
    assert ref.init_from_depth(cams, td, tn, 0) == orc.init_from_depth(cams, td, tn, 0) == -1
    z = np.zeros_like(td)
    assert ref.init_from_depth(cams, z, tn, 5) == orc.init_from_depth(cams, z, tn, 5) == -2
