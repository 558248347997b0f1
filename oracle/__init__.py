"""TEST INFRASTRUCTURE: the CPU parity oracle (see oracle/vp_oracle.h). Never product code."""
