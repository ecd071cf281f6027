// kernels for n_params = 16 (harmonics = 7)
#include "bwm_variants.cuh"

BWM_DEFINE_PICK(16)
BWM_DEFINE_PICK_MASKED(16)
BWM_DEFINE_PICK_MMA(16)
