// sdtw_dp_pick.h -- kernel selection across the instantiation units.
#pragma once
#include "sdtw_dp.cuh"

namespace sdtw {
typedef void (*DpKernel)(DpParams);
DpKernel pick_dp_c1(int WC, bool fma, bool cl);
DpKernel pick_dp_c1t(int WC, bool fma, bool cl);
DpKernel pick_dp_c2(int WC, bool fma, bool cl);
DpKernel pick_dp_c2t(int WC, bool fma, bool cl);
DpKernel pick_dp_c4(int WC, bool fma, bool cl);
DpKernel pick_dp_c4t(int WC, bool fma, bool cl);
DpKernel pick_dpq_c1(int WC, bool fma, bool trace);
DpKernel pick_dpq_c2(int WC, bool fma, bool trace);
DpKernel pick_dp16(int WC);
DpKernel pick_dp8(int WC, bool prune);      // uint8 codebook (sdtw_dp8.cu)
DpKernel pick_dp_c2xs(int WC, bool fma);
DpKernel pick_dp_c2xg(int WC, bool fma);            // query rows in global memory
DpKernel pick_dp_c2ck(int WC, bool fma, int xs);    // + round checkpoints (sdtw_dp_c2k.cu)
inline DpKernel pick_dp(int C, int WC, bool fma, bool trace, bool cl) {
    switch (C) {
        case 1: return trace ? pick_dp_c1t(WC, fma, cl) : pick_dp_c1(WC, fma, cl);
        case 2: return trace ? pick_dp_c2t(WC, fma, cl) : pick_dp_c2(WC, fma, cl);
        case 4: return trace ? pick_dp_c4t(WC, fma, cl) : pick_dp_c4(WC, fma, cl);
        default: return nullptr;
    }
}
}  // namespace sdtw
