"""CPU checks of the single-fluid body-force EXTENSION in the oracle port
(the reference has no single-fluid forcing, so parity is unpinned and the
checks are physical): F = 0 is the reference bit for bit; with F, mass is
conserved and the periodic momentum grows by F per node per step."""
import numpy as np
import pytest

from oracle import oracle as O


@pytest.fixture
def port_force(oracle_port):
    yield oracle_port
    oracle_port.set_body_force(0.0, 0.0, 0.0)


def test_zero_force_is_the_reference(port_force, oracle_ref):
    dims = (9, 8, 7)
    f0 = O.random_state("d3q19", dims, 4, np.float64)
    a, b = f0.copy(), f0.copy()
    port_force.set_body_force(0.0, 0.0, 0.0)
    port_force.single_run("d3q19", dims, 1.3, O.closed_box(), a, None, 5, 0)
    oracle_ref.single_run("d3q19", dims, 1.3, O.closed_box(), b, None, 5, 0)
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64))


@pytest.mark.parametrize("lat,dims", [("d2q9", (12, 10, 1)), ("d3q19", (8, 7, 6)), ("d3q27", (6, 6, 5))])
def test_force_moves_periodic_momentum(port_force, lat, dims):
    F = (2e-5, -1e-5, 5e-6 if dims[2] > 1 else 0.0)
    info = O.lattice_info(lat)
    f = O.random_state(lat, dims, 9, np.float64)
    port_force.set_body_force(*F)
    c = info["c"].astype(np.float64)
    m0 = f.sum()
    j0 = c.T @ f.sum(1)
    steps = 20
    port_force.single_run(lat, dims, 1.1, O.periodic(), f, None, steps, 0)
    n = int(np.prod(dims))
    assert abs(f.sum() - m0) <= 1e-11 * n
    dj = c.T @ f.sum(1) - j0
    # velocity shift forcing: each node gains rho F per step (rho ~ 1 here)
    np.testing.assert_allclose(dj[: info["dim"]], np.array(F[: info["dim"]]) * n * steps, rtol=0.1)
