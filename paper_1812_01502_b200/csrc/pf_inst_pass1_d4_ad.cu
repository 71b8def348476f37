// k_pass1 instantiations for d = 4, fully adapted modes (body: pf_inst_pass1.inc).
#define PASS1_D 4
#define PASS1_SV 0
#define PASS1_ADAPTIVE 1
#define PASS1_LAUNCHER launch_pass1_ad_d4
#define PASS1_SPEC_AD(X) X(kPass1Airpf, 1, 6, 4, 2, 6) X(kPass1Weigh, 1, 6, 4, 2, 6) X(kPass1Resample, 1, 6, 4, 2, 6)  // compile-time instances (C4)
#include "pf_inst_pass1.inc"
