// nodes per direction = 8 (polynomial order 7)
#define ESDG_NQ 8
#include "esdg_inst.cuh"
