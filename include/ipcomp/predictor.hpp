// ipcomp/predictor.hpp -- the planner-facing part of the reference's
// proj/include/ipcomp/predictor.hpp: the amplification factor of each interpolator.  The
// predictor itself runs inside the device passes (paper_2502_04093_b200/csrc/numerics.cu).
#ifndef IPCOMP_PREDICTOR_HPP
#define IPCOMP_PREDICTOR_HPP

#include "ipcomp/grid.hpp"

namespace ipcomp {

// infinity norm of the interpolation operator: linear 1/2 + 1/2, cubic 2 (1/16 + 9/16)
inline double amplification(InterpKind k) { return k == InterpKind::cubic ? 1.25 : 1.0; }

}  // namespace ipcomp

#endif
