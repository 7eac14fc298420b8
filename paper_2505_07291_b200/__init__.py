"""B200-native TOPLOC rollout-verification hot path (INTELLECT-2, arXiv:2505.07291)."""
