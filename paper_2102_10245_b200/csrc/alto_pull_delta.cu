// Pull-engine instantiations for one-word delta streams (alto_pull_impl.cuh).
#include "alto_pull_impl.cuh"
namespace alto {
int pull_run_w1_delta(const alto_pull_args* a, const PullStage& S, int order, cudaStream_t s) {
  return pull_run_delta(a, S, order, s);
}
}  // namespace alto
