// Instantiations of the streaming MTTKRP kernel: 1-word keys, f32 output.
#include "alto_stream.cuh"

namespace alto {

int stream_w1_f32(const DevLayout& d, const uint64_t* tab, const StreamParams& P, int vd, int fd,
                   cudaStream_t s) {
  (void)vd;
  (void)fd;
  return by_order<1, float, float, float>(d, tab, P, s);
}

}  // namespace alto
