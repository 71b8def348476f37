// k_stages instantiations for the float2 state payload (body: pf_inst_stages.inc).
#define STAGES_T float2
#define STAGES_LAUNCHER launch_stages_f2
#define STAGES_PRELOADER preload_stages_f2
#define STAGES_SPEC(X)   // no compile-time (K, b) instances
#include "pf_inst_stages.inc"
