// k_stages instantiations for the float4 state payload (body: pf_inst_stages.inc).
#define STAGES_T float4
#define STAGES_LAUNCHER launch_stages_f4
#define STAGES_PRELOADER preload_stages_f4
#define STAGES_SPEC(X) X(6, 6) X(5, 6) X(4, 6) X(3, 6)  // compile-time (K, b) instances (C4; its shards)
#include "pf_inst_stages.inc"
