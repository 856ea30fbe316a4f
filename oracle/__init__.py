"""CPU oracle package -- test infrastructure only (see dynsparse_oracle.py)."""
