// explicit instantiation of the kernels for L = 128 limbs (C = 16, NB = 8)
#include "kernels.cuh"

namespace mpb {
template struct Launch<16, 8>;
}
