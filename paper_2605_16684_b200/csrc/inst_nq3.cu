// nodes per direction = 3 (polynomial order 2)
#define ESDG_NQ 3
#include "esdg_inst.cuh"
