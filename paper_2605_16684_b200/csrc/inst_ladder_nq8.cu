// Ladder rungs of the volume kernel below the product, NQ = 8 (esdg_inst.cuh).
#define ESDG_NQ 8
#define ESDG_INST_LADDER
#include "esdg_inst.cuh"
