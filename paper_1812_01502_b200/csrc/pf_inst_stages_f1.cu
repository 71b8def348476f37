// k_stages instantiations for the float state payload (body: pf_inst_stages.inc).
#define STAGES_T float
#define STAGES_LAUNCHER launch_stages_f1
#define STAGES_PRELOADER preload_stages_f1
#define STAGES_SPEC(X) X(7, 5) X(6, 5)  // compile-time (K, b) instances (C3)
#include "pf_inst_stages.inc"
