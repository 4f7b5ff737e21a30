// The "widesp" stage-1 layout (16 warps, one CTA per SM; warp-specialised
// fused pass: 8 compute warps with sixteen rows each and setmaxnreg-grown
// registers, 8 copy warps): band.cu compiled a fourth time.
#define EIGENID_STAGE1_NS widesp
#define EIGENID_STAGE1_WIDE 1
#define EIGENID_STAGE1_RW 2
#define EIGENID_STAGE1_SP 1
#include "band.cu"
