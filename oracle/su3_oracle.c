/* C oracle for the SU(3) hot path -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
 * Build: make -C oracle   (gcc -O2 -fopenmp -ffp-contract=off -fno-fast-math)
 */
#include <stdint.h>

#define REAL float
#define SFX f32
#include "su3_oracle_body.h"
#undef REAL
#undef SFX

#define REAL double
#define SFX f64
#include "su3_oracle_body.h"
#undef REAL
#undef SFX
