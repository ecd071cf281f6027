// kernels for n_params = 8 (harmonics = 3)
#include "bwm_variants.cuh"

BWM_DEFINE_PICK(8)
BWM_DEFINE_PICK_MASKED(8)
BWM_DEFINE_PICK_MMA(8)
