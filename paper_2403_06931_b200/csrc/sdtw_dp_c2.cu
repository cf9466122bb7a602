// sdtw_dp_c2.cu -- instantiations of the DP kernel with 2 chain(s) per lane
// (separate translation unit so the kernel variants compile in parallel).
#include "sdtw_dp_pick.h"

namespace sdtw {
template <int WC>
static DpKernel pick_w(bool fma, bool trace, bool cl) {
    if (fma) {
        if (trace) return cl ? sdtw_dp_kernel<2, WC, true, true, true> : sdtw_dp_kernel<2, WC, true, true, false>;
        return cl ? sdtw_dp_kernel<2, WC, true, false, true> : sdtw_dp_kernel<2, WC, true, false, false>;
    }
    if (trace) return cl ? sdtw_dp_kernel<2, WC, false, true, true> : sdtw_dp_kernel<2, WC, false, true, false>;
    return cl ? sdtw_dp_kernel<2, WC, false, false, true> : sdtw_dp_kernel<2, WC, false, false, false>;
}

DpKernel pick_dp_c2(int WC, bool fma, bool trace, bool cl) {
    switch (WC) {
        case 3: return pick_w<3>(fma, trace, cl);
        case 7: return pick_w<7>(fma, trace, cl);
        case 15: return pick_w<15>(fma, trace, cl);
        case 31: return pick_w<31>(fma, trace, cl);
        default: return nullptr;
    }
}
}  // namespace sdtw
