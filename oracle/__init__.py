"""ORACLE / TEST INFRASTRUCTURE ONLY (see oracle/dwdp_oracle.h)."""
