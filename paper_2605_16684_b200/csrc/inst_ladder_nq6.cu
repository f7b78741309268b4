// Ladder rungs of the volume kernel below the product, NQ = 6 (esdg_inst.cuh).
#define ESDG_NQ 6
#define ESDG_INST_LADDER
#include "esdg_inst.cuh"
