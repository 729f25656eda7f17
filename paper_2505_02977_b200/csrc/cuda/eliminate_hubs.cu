// K3's instance with the cooperative wide-column path (hub graphs): the
// kernel source of eliminate.cu compiled as relocatable device code so that
// it can call hub.cu (see launch_eliminate in eliminate.cu).
#define K3_HUBS 1
#include "eliminate.cu"
