// explicit instantiation of the kernels for L = 64 limbs (C = 16, NB = 4)
#include "kernels.cuh"

namespace mpb {
template struct Launch<16, 4>;
}
