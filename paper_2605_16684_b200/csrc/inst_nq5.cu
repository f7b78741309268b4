// nodes per direction = 5 (polynomial order 4)
#define ESDG_NQ 5
#include "esdg_inst.cuh"
