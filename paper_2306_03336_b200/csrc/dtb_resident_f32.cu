// fp32 instantiation of the resident kernel family (dtb_resident.cuh).
#include "dtb_resident.cuh"
template int dtb::launch_resident<float>(const Plan&, const Geometry&, const float*, float*,
                                         int64_t, int, int, const float*, int64_t, bool,
                                         cudaStream_t, unsigned long long*);
