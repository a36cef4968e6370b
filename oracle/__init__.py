"""CPU parity oracle — TEST INFRASTRUCTURE ONLY (see tve_oracle.hpp)."""
