"""B200-native DIC bitmap support count (placeholder; API layer below)."""
