// sdtw_dp8.cu -- instantiations of the uint8-codebook integer DP kernel (SURVEY NEXT-3,
// sdtw_q8.cuh): without pruning and with INF pruning of far cells.  W = 14 (default) and 30:
// an int32 chain value per register doubles the row registers of the half kernel; W = 62 spills.
#include "sdtw_dp_pick.h"
#include "sdtw_q8.cuh"

namespace sdtw {
DpKernel pick_dp8(int WC, bool prune) {
    switch (WC) {
        case 7: return prune ? sdtw_dp2_kernel<Q8Arith<true>, 7> : sdtw_dp2_kernel<Q8Arith<false>, 7>;
        case 15: return prune ? sdtw_dp2_kernel<Q8Arith<true>, 15> : sdtw_dp2_kernel<Q8Arith<false>, 15>;
        default: return nullptr;
    }
}
}  // namespace sdtw
