// The "wide8" stage-1 layout (8 warps, one CTA per SM, sixteen rows per warp
// in the fused pass, up to 255 registers): band.cu compiled a third time.
#define EIGENID_STAGE1_NS wide8
#define EIGENID_STAGE1_WIDE 1
#define EIGENID_STAGE1_RW 2
#include "band.cu"
