// Kernels for d = 1 (see sa_core.cu).
#define SA_D 1
#include "sa_core.cu"
