// sdtw_dpq_c1.cu -- instantiations of the dual-query DP kernel, 1 chain(s) per lane.
#include "sdtw_dp_pick.h"
#include "sdtw_dpq.cuh"

namespace sdtw {
template <int WC>
static DpKernel pick_w(bool fma, bool trace) {
    if (fma) return trace ? sdtw_dpq_kernel<1, WC, true, true> : sdtw_dpq_kernel<1, WC, true, false>;
    return trace ? sdtw_dpq_kernel<1, WC, false, true> : sdtw_dpq_kernel<1, WC, false, false>;
}

DpKernel pick_dpq_c1(int WC, bool fma, bool trace) {
    switch (WC) {
        case 7: return pick_w<7>(fma, trace);
        case 15: return pick_w<15>(fma, trace);
        default: return nullptr;
    }
}
}  // namespace sdtw
