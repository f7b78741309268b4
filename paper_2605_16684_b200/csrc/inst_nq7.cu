// nodes per direction = 7 (polynomial order 6)
#define ESDG_NQ 7
#include "esdg_inst.cuh"
