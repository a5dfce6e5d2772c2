// fp64 instantiation of the resident kernel family (dtb_resident.cuh).
#include "dtb_resident.cuh"
template int dtb::launch_resident<double>(const Plan&, const Geometry&, const double*, double*,
                                          int64_t, int, int, const double*, int64_t, bool,
                                          cudaStream_t, unsigned long long*);
