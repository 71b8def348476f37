// k_pass1 instantiations for d = 4, fully adapted modes (body: pf_inst_pass1.inc).
#define PASS1_D 4
#define PASS1_SV 0
#define PASS1_ADAPTIVE 1
#define PASS1_LAUNCHER launch_pass1_ad_d4
#define PASS1_SPEC_AIR(X) X(1, 6, 4, 2, 6)  // compile-time instances of the AIRPF pass (C4)
#include "pf_inst_pass1.inc"
