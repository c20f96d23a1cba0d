"""B200-native delayed-assembly hot path."""
