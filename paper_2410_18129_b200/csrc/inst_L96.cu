// explicit instantiation of the kernels for L = 96 limbs (C = 16, NB = 6)
#include "kernels.cuh"

namespace mpb {
template struct Launch<16, 6>;
}
