// fp64 instantiation of the pipelined streaming kernel family (dtb_pipe.cuh),
// plus the debug pipe-probe entry point.
#include "dtb_pipe.cuh"

template int dtb::launch_pipe<double>(const Plan&, const Geometry&, const double*, double*,
                                      int64_t, int, int, const double*, int64_t, cudaStream_t,
                                      unsigned long long*);
template int dtb::launch_pipe_wave<double>(const Plan&, const Geometry&, const Geometry&,
                                        const double*, double*, int64_t, int, int, const double*,
                                        int64_t, int64_t, cudaStream_t, unsigned long long*,
                                        const PipeWaveHooks&);

// debug builds (-DDTB_PIPE_PROBE=1): per pipe stage {wait_in, wait_out, total}
// SM cycles, summed over warps since the last call (fp64 kernels); resets
extern "C" int dtb_debug_pipe_probe(uint64_t* out) {
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
