// Kernels for d = 2 (see sa_core.cu).
#define SA_D 2
#include "sa_core.cu"
