"""CPU tier: host geometry of the SPH coupling layer (contact points for the
contact_point pressure model, §6.3); the integrals are GPU-only."""
import numpy as np

from paper_2507_21686_b200 import coupling as C


def test_contact_points_geometry():
    tri = np.array([[0.0, 0.0, 1.0, 0.0, 0.0, 1.0], [0.0, 0.0, 0.0, 1.0, 1.0, 0.0]])  # CCW and CW
    P = np.array([[0.2, 0.2], [-1.0, -1.0], [1.0, 1.0], [0.5, -0.5], [0.0, 0.5]])
    for t in range(2):
        pl = np.array([[i, t] for i in range(P.shape[0])])
        x = C.contact_points(pl, P, tri)
        np.testing.assert_allclose(x, [[0.2, 0.2], [0.0, 0.0], [0.5, 0.5], [0.5, 0.0], [0.0, 0.5]], atol=1e-15)
