// filter_tma.cu — tiled sm_100a ApplyFilter kernel (TMA plane pipeline).
// Placeholder: the tiled kernel lands in the next commit.
#include "common.cuh"
#include "dispatch.h"

namespace vkt {

bool tma_supported(const vkt_filter_args&) { return false; }

int launch_filter_tma(const FilterPlan&, cudaStream_t) { return -1; }

}  // namespace vkt
