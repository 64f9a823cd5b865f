"""TEST INFRASTRUCTURE ONLY: the parity oracle.

`oracle.pyoracle` binds two CPU libraries through ctypes:
  * oracle/build/libssj_oracle.so -- the plain-C restatement (oracle/ssj_oracle.c);
  * oracle/_ref/libssjref.so      -- the UNMODIFIED reference headers compiled through
                                     oracle/ref_shim.cpp (only where the reference exists
                                     or the prebuilt .so travelled with the repo).
Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may import this
package. The product (paper_1812_09141_b200) never does.
"""
