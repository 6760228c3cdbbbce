"""B200-native batched BF-IO step engine (arXiv 2601.17855 hot path)."""
