// Kernel instantiations for the random_waypoints scenario.
#define MRSIM_TASK_ID MRSIM_TASK_RANDOM_WAYPOINTS
#include "step_instantiate.cuh"
