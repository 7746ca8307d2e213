"""B200-native TAPS cost-tensor engine (arXiv 2301.04285 hot path)."""
