"""B200-native SU(3) lattice hot path (arXiv 1309.0551 routines on sm_100a)."""
