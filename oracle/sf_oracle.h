/*
 * sf_oracle.h — plain-C restatement of the reference hot path. TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load this library
 * (as a checker). It is never part of the product path.
 *
 * The entry points have the signatures of include/sf_gpu.h with the prefix sfo_ instead of sf_
 * (same structs, same status codes), so the Python test-suite drives the oracle, the CUDA
 * library and the reference build (oracle/_ref, prefix sfref_) through one API.
 *
 * Pinning: the restatement is checked bit-for-bit against the unmodified reference built in
 * oracle/_ref (tests/test_oracle_cpu.py) and against the reference's own known-answer tests
 * restated in that file. Numerics: FP64, left-to-right evaluation order of the Eigen-API
 * shim (oracle/shim/Eigen/Dense), compiled with -ffp-contract=off.
 */
#ifndef SF_ORACLE_H
#define SF_ORACLE_H

#include "../include/sf_gpu.h"

#endif
