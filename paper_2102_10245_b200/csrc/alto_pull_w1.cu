// Pull-engine instantiations for 64-bit keys (alto_pull_impl.cuh).
#include "alto_pull_impl.cuh"
namespace alto {
int pull_run_w1(const alto_pull_args* a, const PullStage& S, int order, cudaStream_t s) {
  return pull_run<1>(a, S, order, s);
}
}  // namespace alto
