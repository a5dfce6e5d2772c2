// fp32 instantiation of the pipelined streaming kernel family (dtb_pipe.cuh).
#include "dtb_pipe.cuh"

template int dtb::launch_pipe<float>(const Plan&, const Geometry&, const float*, float*,
                                     int64_t, int, int, const float*, int64_t, cudaStream_t,
                                     unsigned long long*);
template int dtb::launch_pipe_wave<float>(const Plan&, const Geometry&, const Geometry&,
                                        const float*, float*, int64_t, int, int, const float*,
                                        int64_t, int64_t, cudaStream_t, unsigned long long*,
                                        const PipeWaveHooks&);

// debug builds (-DDTB_PIPE_PROBE=1): the fp32 kernels' per-stage counters
// (dtb_debug_pipe_probe reads the fp64 ones); resets
extern "C" int dtb_debug_pipe_probe_f32(uint64_t* out) {
#if DTB_PIPE_PROBE
  unsigned long long h[8][3];
  if (cudaMemcpyFromSymbol(h, dtb::g_pipe_probe, sizeof h) != cudaSuccess) return DTB_ECUDA;
  for (int i = 0; i < 24; ++i) out[i] = (&h[0][0])[i];
  unsigned long long z[8][3] = {};
  if (cudaMemcpyToSymbol(dtb::g_pipe_probe, z, sizeof z) != cudaSuccess) return DTB_ECUDA;
  return DTB_OK;
#else
  (void)out;
  return DTB_EINVAL;
#endif
}
