// nodes per direction = 2 (polynomial order 1)
#define ESDG_NQ 2
#include "esdg_inst.cuh"
