// sdtw_dp_c2.cu -- instantiations of the DP kernel with 2 chain(s) per lane, cost/end
// (one translation unit per variant family so they compile in parallel).
#include "sdtw_dp_pick.h"

namespace sdtw {
template <int WC>
static DpKernel pick_w(bool fma, bool cl) {
    if (fma) return cl ? sdtw_dp_kernel<2, WC, true, false, true> : sdtw_dp_kernel<2, WC, true, false, false>;
    return cl ? sdtw_dp_kernel<2, WC, false, false, true> : sdtw_dp_kernel<2, WC, false, false, false>;
}

DpKernel pick_dp_c2(int WC, bool fma, bool cl) {
    switch (WC) {
        case 7: return pick_w<7>(fma, cl);
        case 15: return pick_w<15>(fma, cl);
        default: return nullptr;
    }
}
// single-row query layout (long queries, see smem_layout): cost/end, no cluster
DpKernel pick_dp_c2xs(int WC, bool fma) {
    if (WC != 15) return nullptr;
    return fma ? sdtw_dp_kernel<2, 15, true, false, false, true> : sdtw_dp_kernel<2, 15, false, false, false, true>;
}
// query rows in global memory (XG: long queries, see smem_layout): cost/end, no cluster
DpKernel pick_dp_c2xg(int WC, bool fma) {
    if (WC != 15) return nullptr;
    return fma ? sdtw_dp_kernel<2, 15, true, false, false, false, false, true>
               : sdtw_dp_kernel<2, 15, false, false, false, false, false, true>;
}
}  // namespace sdtw
