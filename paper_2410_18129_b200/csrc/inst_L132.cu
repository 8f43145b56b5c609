// explicit instantiation of the kernels for L = 132 limbs (C = 12, NB = 11)
#include "kernels.cuh"

namespace mpb {
template struct Launch<12, 11>;
}
