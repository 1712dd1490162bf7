// placeholder: replaced by the fused head_dim-128 kernels
#include "kernels.h"
namespace kvc {
bool fast128_applicable(const Geo&) { return false; }
cudaError_t launch_encode_fast128(const EncArgs&, int, cudaStream_t) { return cudaErrorNotSupported; }
cudaError_t launch_decode_fast128(const DecArgs&, int, cudaStream_t) { return cudaErrorNotSupported; }
}
