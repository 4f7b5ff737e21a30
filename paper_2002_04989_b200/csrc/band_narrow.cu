// band_narrow.cu — stage 1 in the "narrow" layout (8 warps, two CTAs per SM,
// 64-row blocks), compiled from band.cu into namespace eigenid_b200::narrow;
// api.cu uses it below the wide-layout size threshold.
#define EIGENID_STAGE1_WIDE 0
#define EIGENID_STAGE1_NS narrow
#include "band.cu"
