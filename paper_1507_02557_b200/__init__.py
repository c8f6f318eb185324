"""hybridwave_b200: B200-native (sm_100a) DG acoustic RHS + time update on
hybrid hex/wedge/pyramid/tet meshes — a drop-in for the hot path of the
reference package ``hybridwave`` (arXiv 1507.02557)."""

__version__ = "0.1.0"
