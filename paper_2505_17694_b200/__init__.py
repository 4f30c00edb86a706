"""B200-native prefix-shared decode attention (CoDec hot path)."""
