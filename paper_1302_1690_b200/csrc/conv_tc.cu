// conv_tc.cu — tcgen05 implicit-GEMM convolutions (placeholder until the kernels land).
#include "conv_tc.h"

namespace mpf {

bool tc_supported(int, int, int) { return false; }
cudaError_t launch_conv_tc(const TcConvArgs&, cudaStream_t) { return cudaErrorNotSupported; }
cudaError_t launch_wgrad_tc(const TcWgradArgs&, int*, cudaStream_t) { return cudaErrorNotSupported; }

}  // namespace mpf
