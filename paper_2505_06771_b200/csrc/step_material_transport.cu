// Kernel instantiations for the material_transport scenario.
#define MRSIM_TASK_ID MRSIM_TASK_MATERIAL_TRANSPORT
#include "step_instantiate.cuh"
