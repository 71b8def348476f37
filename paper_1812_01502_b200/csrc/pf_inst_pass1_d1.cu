// k_pass1 instantiations for d = 1, fused mode (body: pf_inst_pass1.inc).
#define PASS1_D 1
#define PASS1_SV 1
#define PASS1_ADAPTIVE 0
#define PASS1_LAUNCHER launch_pass1_d1
#define PASS1_SPEC(X) X(2, 5, 6, 2, 2)  // compile-time instances of the fused pass (C3)
#include "pf_inst_pass1.inc"
