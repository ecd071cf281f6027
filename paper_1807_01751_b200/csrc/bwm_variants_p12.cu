// kernels for n_params = 12 (harmonics = 5)
#include "bwm_variants.cuh"

BWM_DEFINE_PICK(12)
BWM_DEFINE_PICK_MASKED(12)
BWM_DEFINE_PICK_MMA(12)
