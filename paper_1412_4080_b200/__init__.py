"""B200-native dynamic-screening solver (arXiv 1412.4080 hot path)."""
