// placeholder: replaced by the tcgen05 similarity kernel
#include "kernels.h"
namespace kvf {
bool tc_supported(const SimArgs& a, const char** why) { *why = "not built"; return false; }
cudaError_t launch_sim_tc(const SimArgs& a, cudaStream_t s) { return cudaErrorNotSupported; }
}
