// Instantiations of the specialised streaming MTTKRP: 1-word keys, f32 output.
#include "alto_mstream.cuh"

namespace alto {

int fast_w1_f32(const DevLayout& d, const uint64_t* tab, const StreamParams& P, int vd, int fd, cudaStream_t s) {
  if (vd == ALTO_F32 && fd == ALTO_F32) return try_fast<1, float, float>(d, tab, P, s);
  return ALTO_EUNSUPPORTED;
}

}  // namespace alto
