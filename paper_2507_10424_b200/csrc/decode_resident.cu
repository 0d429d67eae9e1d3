// decode_resident.cu -- SMEM-resident persistent schedule (placeholder until implemented).
#include "ldpc_internal.cuh"

namespace ldpc {

ResidentPlan plan_resident(const HostGraph &g, bool loc16, int device) {
    (void)g; (void)loc16; (void)device;
    return ResidentPlan{};
}

int launch_resident(const Graph &, const ResidentPlan &, const float *, int64_t, int, bool, bool, bool, float *,
                    uint8_t *, int32_t *, uint8_t *, unsigned long long *, int *, cudaStream_t) {
    return 0;
}

}  // namespace ldpc
