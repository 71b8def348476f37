// k_stages instantiations for the float state payload (body: pf_inst_stages.inc).
#define STAGES_T float
#define STAGES_LAUNCHER launch_stages_f1
#include "pf_inst_stages.inc"
