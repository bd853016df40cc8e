/* rp_oracle_q.c -- the oracle's pair program and exhaustive search in IEEE binary128.
 *
 * TEST INFRASTRUCTURE ONLY (see rp_oracle.h).  Same source as the long double instance
 * (rp_oracle_pair.inc), instantiated with REAL = __float128 (gcc soft-float, libgcc; no libm
 * call is needed: the transform scales by an exact power of two).
 */
#include "rp_oracle.h"

#include <math.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define REAL __float128
#define RABS(x) ((x) < 0 ? -(x) : (x))
#define RFINITE(x) ((x) == (x) && (x) - (x) == 0)
#define ORC_PFX(name) name##_q
#include "rp_oracle_pair.inc"
