// Instantiations of the streaming MTTKRP kernel: 2-word keys, f32 output.
#include "alto_stream.cuh"

namespace alto {

int stream_w2_f32(const DevLayout& d, const uint64_t* tab, const StreamParams& P, int vd, int fd,
                   cudaStream_t s) {
  (void)vd;
  (void)fd;
  return by_order<2, float, float, float>(d, tab, P, s);
}

}  // namespace alto
