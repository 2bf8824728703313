"""CPU checker package (test infrastructure only)."""
