// fp32 instantiation of the pipelined streaming kernel family (dtb_pipe.cuh).
#include "dtb_pipe.cuh"

template int dtb::launch_pipe<float>(const Plan&, const Geometry&, const float*, float*,
                                     int64_t, int, int, const float*, int64_t, cudaStream_t,
                                     unsigned long long*);
template int dtb::launch_pipe_wave<float>(const Plan&, const Geometry&, const Geometry&,
                                        const float*, float*, int64_t, int, int, const float*,
                                        int64_t, int64_t, cudaStream_t, unsigned long long*,
                                        const PipeWaveHooks&);
