// The f16 unit of the BN kernels: cgbn.cu compiled for one activation dtype (see there).
#define CGBN_TU_ACT 2
#include "cgbn.cu"
