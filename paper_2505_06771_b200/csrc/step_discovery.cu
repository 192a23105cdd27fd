// Kernel instantiations for the discovery scenario.
#define MRSIM_TASK_ID MRSIM_TASK_DISCOVERY
#include "step_instantiate.cuh"
