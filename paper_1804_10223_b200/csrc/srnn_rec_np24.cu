// Instantiation of the persistent recurrent kernel for NP = 24 register slots
// per lane (split per NP so nvcc can compile instances in parallel).
#include "srnn_recurrent.cuh"
namespace srnn {
template int launch_np<24>(int, int, const RecParams&, int, size_t, void*, bool, int*, int*);
}
