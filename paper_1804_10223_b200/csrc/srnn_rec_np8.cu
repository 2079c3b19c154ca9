// Instantiations of the persistent recurrent kernel for NP = 8 register slots
// per lane (one file per NP so nvcc compiles instances in parallel).
#include "srnn_recurrent.cuh"
namespace srnn {
template int launch_np<8, false>(int, int, const RecParams&, int, size_t, void*, bool, int*, int*);
template int launch_np<8, true>(int, int, const RecParams&, int, size_t, void*, bool, int*, int*);
}
