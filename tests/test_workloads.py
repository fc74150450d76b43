"""The shared input generator (splitmix64 contract)."""
import numpy as np

from workloads import splitmix64, uniform, make_u0, config, CONFIGS


def test_splitmix64_reference_values():
    # Published splitmix64 outputs for seed 0 (Vigna's reference splitmix64.c).
    z = splitmix64(0, 3)
    assert [int(v) for v in z] == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]


def test_uniform_range_and_determinism():
    a = uniform(5, 10000, -0.05, 0.05)
    assert a.min() >= -0.05 and a.max() < 0.05
    assert np.array_equal(a, uniform(5, 10000, -0.05, 0.05))
    assert abs(a.mean()) < 2e-3


def test_config_geometry():
    assert config("c1").nx == 64 and config("c1").ny == 1
    assert config("c2").nx == 1024
    assert config("c3").nx == 511 and config("c3").ny == 511
    assert config("c4").nx == 257
    assert config("c5").nx == 2049 and config("c5").dofs == 2049 * 2049 * 512
    for p in CONFIGS.values():
        assert p.theta == 1.0


def test_u0_shapes():
    for name in ("c1", "c2", "c3", "c4"):
        p = config(name)
        u0 = make_u0(p)
        assert u0.shape == (p.ny, p.nx)
    u = make_u0(config("c1"))
    assert abs(u[0, 31] - np.sin(np.pi * 32 / 65)) == 0.0
