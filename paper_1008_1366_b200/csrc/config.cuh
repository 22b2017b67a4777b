// config.cuh -- every tuning knob of the library in one table (compile-time
// defaults; tools/build_variant.sh rebuilds the library with -D overrides for
// A/B runs).  Each value below was chosen by an A/B measurement on B200
// (profiles/r01_ab/, profiles/r02/ab/); the comment next to the use site
// gives the numbers.  Two knobs are read from the environment at run time
// (slab grouping of the 3D calls, nd.cu): IDC_SLAB_L2_FRAC, IDC_SLAB_STREAMS.
//
// | knob                    | default | what it selects                                                        |
// |-------------------------|---------|------------------------------------------------------------------------|
// | IDC_PDL                 | 1       | kernels launched with programmatic dependent launch (pdl.cuh)          |
// | IDC_PDL_TRIGGER         | 0       | early griddepcontrol.launch_dependents at kernel start (pdl.cuh)       |
// | IDC_FOLD_TW             | 1       | Stockham pass twiddles folded into FMA-form DIT butterflies (fft_dev.cuh) |
// | IDC_ROWS_TW_COH_MIN_E   | 16      | row kernels with E >= this reload pass twiddles per pass (coherent loads) |
// | IDC_V2_MAX_M            | 4096    | rows up to this m run the rows2.cu kernels (K2/K3/K4 register-resident) |
// | IDC_V3_MIN_M            | 512     | hconv / tconv rows from this m run the TMA-staged rows3.cu K3/K4        |
// | IDC_ROWS_E              | 16      | rows2.cu elements per thread for m >= 1024                             |
// | IDC_ROWS_CTA_THREADS    | 256     | rows2.cu threads per CTA                                                |
// | IDC_ROWS_REGS           | 255     | rows2.cu register budget per thread (CTAs per SM = 64K / (threads*regs)) |
// | IDC_ROWS_PREFETCH       | 1       | rows2.cu: L2 bulk prefetch of the next rows (unstaged m)               |
// | IDC_ROWS2_TMA_MAX       | 512     | K2 stages f, g rows in shared memory (bulk copies) up to this m         |
// | IDC_K2_PARK_MIN         | 4096    | K2 parks the r = 0 result in shared memory from this m                  |
// | IDC_K2_ONE_READ         | 1       | K2 (E = 8, staged rows) builds both residues' streams from one read     |
// | IDC_K3_ONE_SPLIT_MAXE   | 16      | K3 splits all three residues from one staged read up to this E          |
// | IDC_K3_STAGGER_MAX_M    | 512     | K3 runs its transforms as staggered pairs (fft2s, two exchange buffers) |
// | IDC_K3_STAGE_AS_XB      | 2048    | K3 from this m: first transform pair staggered in the consumed stage    |
// | IDC_ROWS3_E8_MAX        | 512     | rows3.cu (K3/K4) use E = 8 up to this m, E = 16 above                   |
// | IDC_K2_G512             | 4       | rows2.cu row groups (64-thread rows) per CTA at m = 512 (K2)            |
// | IDC_K3_G512 / K4_G512   | 6 / 4   | K3 / K4 row groups (64-thread rows) per CTA at m <= 512                 |
// | IDC_ROWS3_MINB_SMALL    | 1       | rows3.cu CTAs per SM for m <= 512                                       |
// | IDC_PENCIL_TMA          | 1       | 2D/3D pencils use the TMA kernels of pencils2.cu for 64 <= m <= 4096    |
// | IDC_PENCIL_E            | 8       | pencils2.cu elements per thread where not specialised                  |
// | IDC_PENCIL_THREADS      | 512     | pencils2.cu threads per CTA where not specialised                      |
// | IDC_PENCIL_MINB         | 1       | pencils2.cu CTAs per SM (register cap)                                  |
// | IDC_PENCIL0_THREADS     | =above  | K7 threads per CTA where not specialised                               |
// | IDC_PENCIL0_MINB        | =above  | K7 CTAs per SM                                                          |
// | IDC_K56_NARROW_MIN/MAX  | 256/1024| K5/K6 with 128-thread CTAs (half-width tiles) for m in this range      |
// | IDC_K56_TMA_STORE_MAXW  | 2       | K5/K6 store tiles of at most this many columns by TMA tensor stores     |
// | IDC_K5_PAIR             | 1       | K5 with per-thread stores: odd/even streams as a staggered pair (fft2s) |
// | IDC_K5_DOUBLE_XB        | 1       | K5 second exchange buffer (odd stream's store drains during the even)  |
// | IDC_K78_WIDE_MIN/MAX    | 256/4096| K7/K8 with E = 16 and 256-thread CTAs for m in this range               |
// | IDC_K78_NARROW_MASK     | m=1024,256 | K7/K8 with 128-thread CTAs for the m whose log2 bit is set           |
// | IDC_K7_TMA_STORE        | 1       | K7 residue tiles leave through the exchange buffer by TMA stores        |
// | IDC_K7_KEEP_RAW         | 1       | K7 reads U_k, U_{k-m} once into registers; next tile loaded at once     |
// | IDC_K8_TMA_STORE        | 2       | K8: both output halves by TMA stores (1: U_k only, 0: per thread)      |
// | IDC_PENCIL_WAIT_IN_FFT  | 1       | K7/K8 wait for the previous TMA store's read of xb after the first     |
// |                         |         | radix pass of the next FFT (0: before the FFT)                          |
#pragma once

#ifndef IDC_FOLD_TW
#define IDC_FOLD_TW 1
#endif
#ifndef IDC_ROWS_TW_COH_MIN_E
#define IDC_ROWS_TW_COH_MIN_E 16
#endif

#ifndef IDC_V2_MAX_M
#define IDC_V2_MAX_M 4096
#endif
#ifndef IDC_V3_MIN_M
#define IDC_V3_MIN_M 512
#endif
#ifndef IDC_ROWS_E
#define IDC_ROWS_E 16
#endif
#ifndef IDC_ROWS_CTA_THREADS
#define IDC_ROWS_CTA_THREADS 256
#endif
#ifndef IDC_ROWS_REGS
#define IDC_ROWS_REGS 255
#endif
#ifndef IDC_ROWS_PREFETCH
#define IDC_ROWS_PREFETCH 1
#endif
#ifndef IDC_ROWS2_TMA_MAX
#define IDC_ROWS2_TMA_MAX 512
#endif
#ifndef IDC_K2_PARK_MIN
#define IDC_K2_PARK_MIN 4096
#endif
#ifndef IDC_K2_ONE_READ
#define IDC_K2_ONE_READ 1
#endif
#ifndef IDC_K3_ONE_SPLIT_MAXE
#define IDC_K3_ONE_SPLIT_MAXE 16
#endif
#ifndef IDC_K3_STAGGER_MAX_M
#define IDC_K3_STAGGER_MAX_M 512
#endif
#ifndef IDC_K3_STAGE_AS_XB
#define IDC_K3_STAGE_AS_XB 2048
#endif
#ifndef IDC_ROWS3_E8_MAX
#define IDC_ROWS3_E8_MAX 512
#endif
#ifndef IDC_K2_G512
#define IDC_K2_G512 4
#endif
#ifndef IDC_K3_G512
#define IDC_K3_G512 6
#endif
#ifndef IDC_K4_G512
#define IDC_K4_G512 4
#endif
#ifndef IDC_ROWS3_MINB_SMALL
#define IDC_ROWS3_MINB_SMALL 1
#endif
#ifndef IDC_PENCIL_TMA
#define IDC_PENCIL_TMA 1
#endif
#ifndef IDC_PENCIL_E
#define IDC_PENCIL_E 8
#endif
#ifndef IDC_PENCIL_THREADS
#define IDC_PENCIL_THREADS 512
#endif
#ifndef IDC_PENCIL_MINB
#define IDC_PENCIL_MINB 1
#endif
#ifndef IDC_PENCIL0_THREADS
#define IDC_PENCIL0_THREADS IDC_PENCIL_THREADS
#endif
#ifndef IDC_PENCIL0_MINB
#define IDC_PENCIL0_MINB IDC_PENCIL_MINB
#endif
#ifndef IDC_K56_NARROW_MIN
#define IDC_K56_NARROW_MIN 256
#endif
#ifndef IDC_K56_NARROW_MAX
#define IDC_K56_NARROW_MAX 1024
#endif
#ifndef IDC_K56_TMA_STORE_MAXW
#define IDC_K56_TMA_STORE_MAXW 2
#endif
#ifndef IDC_K5_PAIR
#define IDC_K5_PAIR 1
#endif
#ifndef IDC_K5_DOUBLE_XB
#define IDC_K5_DOUBLE_XB 1
#endif
#ifndef IDC_K78_WIDE_MIN
#define IDC_K78_WIDE_MIN 256
#endif
#ifndef IDC_K78_WIDE_MAX
#define IDC_K78_WIDE_MAX 4096
#endif
#ifndef IDC_K78_NARROW_MASK
#define IDC_K78_NARROW_MASK ((1 << 10) | (1 << 8))
#endif
#ifndef IDC_K7_TMA_STORE
#define IDC_K7_TMA_STORE 1
#endif
#ifndef IDC_K7_KEEP_RAW
#define IDC_K7_KEEP_RAW 1
#endif
#ifndef IDC_K8_TMA_STORE
#define IDC_K8_TMA_STORE 2
#endif
#ifndef IDC_PENCIL_WAIT_IN_FFT
#define IDC_PENCIL_WAIT_IN_FFT 1
#endif
