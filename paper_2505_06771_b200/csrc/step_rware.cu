// Kernel instantiations for the rware scenario.
#define MRSIM_TASK_ID MRSIM_TASK_RWARE
#include "step_instantiate.cuh"
