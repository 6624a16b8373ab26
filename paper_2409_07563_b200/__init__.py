"""B200-native MPPI optimisation iteration (MPPI-Generic, arXiv 2409.07563)."""
