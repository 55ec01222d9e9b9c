"""B200-native dense diffeomorphic matching (FireANTs direct-mode loop)."""
