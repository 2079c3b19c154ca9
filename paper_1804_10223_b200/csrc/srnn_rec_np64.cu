// Instantiations of the persistent recurrent kernel for NP = 64 register slots
// per lane (one file per NP so nvcc compiles instances in parallel).
#include "srnn_recurrent.cuh"
namespace srnn {
template int launch_np<64, false>(int, int, const RecParams&, int, size_t, void*, bool, int*, int*);
template int launch_np<64, true>(int, int, const RecParams&, int, size_t, void*, bool, int*, int*);
}
