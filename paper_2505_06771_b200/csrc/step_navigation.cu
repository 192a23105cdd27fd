// Kernel instantiations for the navigation scenario.
#define MRSIM_TASK_ID MRSIM_TASK_NAVIGATION
#include "step_instantiate.cuh"
