// Kernel instantiations for the foraging scenario.
#define MRSIM_TASK_ID MRSIM_TASK_FORAGING
#include "step_instantiate.cuh"
