// sdtw_dp_pick.h -- kernel selection across the per-C instantiation units.
#pragma once
#include "sdtw_dp.cuh"

namespace sdtw {
typedef void (*DpKernel)(DpParams);
DpKernel pick_dp_c1(int WC, bool fma, bool trace, bool cl);
DpKernel pick_dp_c2(int WC, bool fma, bool trace, bool cl);
DpKernel pick_dp_c4(int WC, bool fma, bool trace, bool cl);
}  // namespace sdtw
