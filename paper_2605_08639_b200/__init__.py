"""B200-native ReLibra MoE-layer hot path (placeholder; API mirror filled in below)."""
