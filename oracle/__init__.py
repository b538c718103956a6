"""CPU oracle -- TEST INFRASTRUCTURE ONLY (see cfp_oracle.h)."""
