// Kernel instantiations for the warehouse scenario.
#define MRSIM_TASK_ID MRSIM_TASK_WAREHOUSE
#include "step_instantiate.cuh"
