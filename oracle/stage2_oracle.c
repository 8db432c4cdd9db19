/*
 * stage2_oracle.c -- CPU ORACLE FOR TESTS.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load or call this library.  The product path
 * (paper_2301_07964_b200/, include/ht_stage2.h) never does, and shares no
 * code, header, table or helper with it.
 *
 * What it computes: stage two of the two-stage Hessenberg-triangular
 * reduction (arxiv 2301.07964, Alg. 2 "Reduction to
 * Hessenberg-triangular form without blocking"): an r-Hessenberg-triangular
 * pencil (A,B) is reduced in place to Hessenberg-triangular
 * form with Q(A_out,B_out)Z^* = (A_in,B_in), one Householder
 * reflector at a time, in plain fp64 (real) or fp64 complex.
 * No blocking, fusion or reordering beyond Alg. 2.  OpenMP only splits each
 * single reflector application over its independent columns (left) or rows
 * (right), each computed by one thread in a fixed order, so results are
 * bitwise independent of the thread count.
 *
 * Pins (tests/test_oracle_*.py, "not gpu"): larfg closed form ([3,4]),
 * RQ reconstruction, r=1 exact identity, n<=2 no-op, an independent
 * Moler-Stewart Givens reduction (tests/givens_ref.py) after phase
 * normalisation, LAPACK gehrd (scipy.linalg.hessenberg) for B = I,
 * backward-error / orthogonality invariants, exact zeros, Fig. 5 structure
 * traces, and the session-derived n=4 worked example
 * (SURVEY.md App. A.5).
 */
#include <complex.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ---- real instantiation ---- */
#define SCALAR double
#define SUFFIX d
#define CONJ(x) (x)
#define REAL(x) (x)
#define IMAG(x) (0.0)
#define ABS2(x) ((x) * (x))
#define FLOPS_PER_FMA 2.0
#include "stage2_oracle_impl.h"
#undef SCALAR
#undef SUFFIX
#undef CONJ
#undef REAL
#undef IMAG
#undef ABS2
#undef FLOPS_PER_FMA

/* ---- complex instantiation ---- */
#define SCALAR double complex
#define SUFFIX z
#define CONJ(x) conj(x)
#define REAL(x) creal(x)
#define IMAG(x) cimag(x)
#define ABS2(x) (creal(x) * creal(x) + cimag(x) * cimag(x))
#define FLOPS_PER_FMA 8.0
#include "stage2_oracle_impl.h"

/* thread control for the cpu_baseline leg (records the count it used) */
int oracle_set_threads(int nthreads)
{
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
    return omp_get_max_threads();
#else
    (void)nthreads;
    return 1;
#endif
}
