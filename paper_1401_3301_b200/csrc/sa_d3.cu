// Kernels for d = 3 (see sa_core.cu).
#define SA_D 3
#include "sa_core.cu"
