// nodes per direction = 6 (polynomial order 5)
#define ESDG_NQ 6
#include "esdg_inst.cuh"
