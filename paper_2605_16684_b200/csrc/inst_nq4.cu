// nodes per direction = 4 (polynomial order 3)
#define ESDG_NQ 4
#include "esdg_inst.cuh"
