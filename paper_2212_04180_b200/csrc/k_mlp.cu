// k_mlp.cu — K4 synthetic-MLP fitness (NUMERICS N14). Placeholder until the tcgen05 kernel lands.
#include <string>

#include "es_internal.h"

namespace esb {
void* mlp_problem_create(const int32_t*, int32_t, int32_t, uint64_t, cudaStream_t,
                         std::string* err) {
  *err = "unsupported: the MLP fitness kernel is not built in this revision";
  return nullptr;
}
void mlp_problem_destroy(void*) {}
int64_t mlp_problem_dims(const void*) { return -1; }
cudaError_t launch_mlp_eval(void*, const float*, int64_t, float*, cudaStream_t) {
  return cudaErrorNotSupported;
}
}  // namespace esb
