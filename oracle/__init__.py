"""CPU oracle of the reference algorithm -- test infrastructure only (see tpf_oracle.py)."""
