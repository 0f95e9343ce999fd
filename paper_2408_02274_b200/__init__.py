"""B200-native IFGF N-Muller matvec (arXiv 2408.02274 hot path)."""
