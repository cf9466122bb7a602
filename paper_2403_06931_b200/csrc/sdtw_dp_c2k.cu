// sdtw_dp_c2k.cu -- the two-chain cost/end kernel with round checkpoints (CKPT): the last
// column of every round is stored for the checkpointed start index.
#include "sdtw_dp_pick.h"

namespace sdtw {
DpKernel pick_dp_c2ck(int WC, bool fma, bool xs) {
    if (WC != 15) return nullptr;
    if (xs) return fma ? sdtw_dp_kernel<2, 15, true, false, false, true, true>
                       : sdtw_dp_kernel<2, 15, false, false, false, true, true>;
    return fma ? sdtw_dp_kernel<2, 15, true, false, false, false, true>
               : sdtw_dp_kernel<2, 15, false, false, false, false, true>;
}
}  // namespace sdtw
