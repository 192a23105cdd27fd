// Kernel instantiations for the predator_prey scenario.
#define MRSIM_TASK_ID MRSIM_TASK_PREDATOR_PREY
#include "step_instantiate.cuh"
