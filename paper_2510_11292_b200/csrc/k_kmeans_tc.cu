// tcgen05/TMEM k-means assignment — placeholder until the tensor-core kernel lands.
#include "lkv_internal.cuh"
namespace lkv {
bool kmeans_tc_available() { return false; }
cudaError_t launch_assign_tc(const KmArgs&, cudaStream_t) { return cudaErrorNotSupported; }
}  // namespace lkv
