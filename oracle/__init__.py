"""CPU oracle (test infrastructure only; see oracle/efem_oracle.cpp header)."""
