/*
 * ooc_emul64.c -- TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * The literal out-of-core emulator of ooc_emul.c in the paper's own
 * precision (fp64; rates 32/64 and 24/64):
 * the same region bookkeeping with fp64 fields, the fp64 codec (zfp_ref64.c)
 * and the fp64 stencil (orc_step_planes_f64).  It pins orc64_advance (the
 * reduced schedule) at rates > 0, as ooc_emul.c pins orc_advance.
 */
#define OOC_REAL double
#define OOC_BYTES orc_zfp_bytes
#define OOC_ENCODE orc64_zfp_encode
#define OOC_DECODE orc64_zfp_decode
#define OOC_STEP_PLANES orc_step_planes_f64
#define OOC_EMULATE orc64_ooc_emulate
#define OOC_NAN nan("")
#include "ooc_emul.c"
