// C ABI entry points (see sa_core.cu).
#define SA_ABI
#include "sa_core.cu"
