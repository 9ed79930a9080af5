"""B200-native batched Simple* nonlinear solvers (drop-in for nlkit's solve path)."""
