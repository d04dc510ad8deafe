// cvk_phased_g4.cu -- the phase kernels of cvk_phased.cu compiled a second
// time with 4 consumer groups of 128 rows per CTA (namespace cvk_g4).  Rows
// with many out-of-chunk gathers (FEM-3D, ~15 nnz/row) keep more rows in
// flight this way: 1M-DOF FEM BiCGSTAB 286 -> 268 us per iteration, tfQMR
// 278 -> 261; the 5-point cavity prefers 2 x 224.  cvk_api.cu picks the
// flavor per matrix (nnz/row > 8, or CVK_STREAM_FLAVOR).
#define CVK_STREAM_GROUPS 4
#define CVK_STREAM_ROWS 128
#define cvk cvk_g4
#include "cvk_phased.cu"
