// k_stages instantiations for the State8 state payload (body: pf_inst_stages.inc).
#define STAGES_T State8
#define STAGES_LAUNCHER launch_stages_f8
#define STAGES_PRELOADER preload_stages_f8
#define STAGES_SPEC(X) X(3, 8) X(2, 8)  // compile-time (K, b) instances (C2)
#include "pf_inst_stages.inc"
