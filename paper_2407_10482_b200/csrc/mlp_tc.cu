// mlp_tc.cu — K2 (tensor mode): placeholder until the tcgen05 kernel lands.
#include "render.cuh"
#include <cstring>
namespace ngprt_dev {
size_t psi_tc_bytes() { return 16; }
void pack_psi_tc(const float*, void* out) { std::memset(out, 0, 16); }
void launch_shade_tensor(const DevScene&, const void*, const RayAcc*, float*, size_t, cudaStream_t) {}
}  // namespace ngprt_dev
