// Kernel instantiations for the arctic_transport scenario.
#define MRSIM_TASK_ID MRSIM_TASK_ARCTIC_TRANSPORT
#include "step_instantiate.cuh"
