"""Test oracle for arXiv 1812.01502 (BPF step with augmented resampling).

TEST INFRASTRUCTURE ONLY -- see oracle/pf_oracle.c header.  Nothing under
paper_1812_01502_b200/ imports this package.
"""
