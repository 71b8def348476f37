// k_pass1 instantiations for d = 2, fully adapted modes (body: pf_inst_pass1.inc).
#define PASS1_D 2
#define PASS1_SV 0
#define PASS1_ADAPTIVE 1
#define PASS1_LAUNCHER launch_pass1_ad_d2
#include "pf_inst_pass1.inc"
