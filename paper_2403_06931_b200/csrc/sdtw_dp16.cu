// sdtw_dp16.cu -- instantiations of the packed-half DP kernel.
#include "sdtw_dp_pick.h"
#include "sdtw_dp2.cuh"

namespace sdtw {
DpKernel pick_dp16(int WC) {
    switch (WC) {
        case 7: return sdtw_dp2_kernel<Half2Arith, 7>;
        case 15: return sdtw_dp2_kernel<Half2Arith, 15>;
        case 31: return sdtw_dp2_kernel<Half2Arith, 31>;
        default: return nullptr;
    }
}
}  // namespace sdtw
