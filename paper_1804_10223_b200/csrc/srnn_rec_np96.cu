// Instantiations of the persistent recurrent kernel for NP = 96 register slots
// per lane; fp16 mode only (one register per pair).
#include "srnn_recurrent.cuh"
namespace srnn {
template int launch_np<96, true>(int, int, const RecParams&, int, size_t, void*, bool, int*, int*);
}
