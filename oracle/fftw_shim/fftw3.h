/* CPU provider of the FFTW3 subset the reference calls (test infrastructure).
 *
 * FFTW3 is not installed in this image; the reference's only
 * FFT call site is gridder.hpp:85-100 (fft3_inplace), reached from
 * ewald.hpp:542,555,569,597.  This header declares exactly the symbols used
 * there -- fftw_complex, fftw_plan, fftw_plan_dft_3d, fftw_execute,
 * fftw_destroy_plan, FFTW_FORWARD/FFTW_BACKWARD, FFTW_ESTIMATE -- with FFTW's
 * published semantics: unnormalised complex-to-complex DFT, row-major
 * [n0][n1][n2] (last index fastest), forward sign -1 (e^{-i}), backward +1.
 *
 * The implementation (fftw_shim.cpp) is a mixed-radix (2/3/4/5 + generic
 * prime) decimation-in-time FFT with exactly computed twiddles, checked
 * against the reference's own FFT contracts (test_gridder.cpp:44-76).
 * It is only ever linked into oracle/_ref (the compiled reference); the
 * product path uses cuFFT.
 */
#ifndef ESP_ORACLE_FFTW3_SHIM_H
#define ESP_ORACLE_FFTW3_SHIM_H

#ifdef __cplusplus
extern "C" {
#endif

typedef double fftw_complex[2];
typedef struct fftw_plan_s* fftw_plan;

#define FFTW_FORWARD (-1)
#define FFTW_BACKWARD (+1)
#define FFTW_MEASURE (0U)
#define FFTW_ESTIMATE (1U << 6)

fftw_plan fftw_plan_dft_3d(int n0, int n1, int n2, fftw_complex* in, fftw_complex* out,
                           int sign, unsigned flags);
void fftw_execute(const fftw_plan p);
void fftw_destroy_plan(fftw_plan p);

#ifdef __cplusplus
}
#endif

#endif
