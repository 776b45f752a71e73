"""CPU oracle of the EM hot path -- test infrastructure only (see einet_oracle)."""
