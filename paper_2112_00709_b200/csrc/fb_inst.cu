// fb_inst.cu — instantiates k_fb<FBX_BWD, FBX_MODE, spt, MAXT> for every
// states-per-thread / CTA-size variant.  Compiled once per (direction, mode)
// with -DFBX_BWD=0|1 -DFBX_MODE=0|1|2|4 so the eight heavy instantiation sets
// build in parallel.
#include "fb_device.cuh"

#if !defined(FBX_BWD) || !defined(FBX_MODE)
#error "compile with -DFBX_BWD=<0|1> -DFBX_MODE=<0|1|2|4>"
#endif

namespace fbx {

template <bool BWD, int MODE, int MAXT>
static KFn pick_spt(int spt) {
    switch (spt) {
        case 1: return k_fb<BWD, MODE, 1, MAXT>;
        case 2: return k_fb<BWD, MODE, 2, MAXT>;
        case 3: return k_fb<BWD, MODE, 3, MAXT>;
        case 4: return k_fb<BWD, MODE, 4, MAXT>;
        case 6: return k_fb<BWD, MODE, 6, MAXT>;
        default: return k_fb<BWD, MODE, 8, MAXT>;
    }
}

// The CTA size T ∈ {128, 256, 512, 1024} is a compile-time constant of the
// kernel (MAXT == T): 128 (seven CTAs per SM), 256 (two per SM), 512 (≤ 128
// registers per thread), 1024.
template <bool BWD, int MODE>
KFn pick_fb(int spt, int T) {
    if (T <= 128) return pick_spt<BWD, MODE, 128>(spt);
    if (T <= 256) return pick_spt<BWD, MODE, 256>(spt);
    if (T <= 512) return pick_spt<BWD, MODE, 512>(spt);
    return pick_spt<BWD, MODE, 1024>(spt);
}

template KFn pick_fb<(bool)FBX_BWD, FBX_MODE>(int, int);

}  // namespace fbx
