/*
 * spidgpu_status.h -- status codes of the spidgpu C ABI.
 *
 * The reference reports failures as spid::Error{name, message}
 * (/root/reference/proj/include/spid/error.hpp:11-24). A C ABI cannot throw,
 * so every entry point returns one of these codes and spidgpu_status_name()
 * maps it back to the reference's exact error name, letting a C++ shim
 * rethrow spid::Error(name, msg) unchanged. Per-subdomain status arrays of
 * the batched calls use the same codes.
 */
#ifndef SPIDGPU_STATUS_H
#define SPIDGPU_STATUS_H

enum spidgpu_status {
    SPID_OK = 0,
    SPID_NON_FINITE_INPUT = 1,  /* "NonFiniteInput"   qr.cpp:35, id.cpp:42 */
    SPID_RANK_UNREACHABLE = 2,  /* "RankUnreachable"  qr.cpp:38,79 */
    SPID_ZERO_MATRIX = 3,       /* "ZeroMatrix"       qr.cpp:51,109 */
    SPID_SINGULAR_PIVOT = 4,    /* "SingularPivot"    qr.cpp:140 */
    SPID_DIMENSION_MISMATCH = 5,/* "DimensionMismatch" qr.cpp:131,133; id.cpp:77,88,94 */
    SPID_NON_FINITE_COEFFS = 6, /* "NonFiniteCoeffs"  id.cpp:26 */
    SPID_BAD_RANK_RULE = 7,     /* "BadRankRule"      qr.hpp:17,23 */
    SPID_EMPTY_MATRIX = 8,      /* "EmptyMatrix"      dense_matrix.hpp:53 */
    SPID_EMPTY_SELECTION = 9,   /* "EmptySelection"   dense_matrix.cpp:72 */
    SPID_INDEX_OUT_OF_RANGE = 10,/* "IndexOutOfRange" dense_matrix.cpp:75 */
    SPID_GEOMETRY_MISMATCH = 11,/* "GeometryMismatch" grid.cpp:138 */
    SPID_ZERO_REFERENCE = 12,   /* "ZeroReference"    metrics.cpp:18-19 */
    SPID_ZERO_DENOMINATOR = 13, /* "ZeroDenominator"  metrics.cpp:6-9 */
    SPID_BAD_SUBSAMPLE_SPEC = 14,/* "BadSubsampleSpec" grid.cpp:65-69 */
    SPID_EMPTY_SKETCH = 15,     /* "EmptySketch"      grid.cpp:78,110 */
    SPID_EXTRAPOLATION_REQUIRED = 16, /* "ExtrapolationRequired" interp.cpp:27-29 */
    SPID_BAD_GRID_GEOM = 17,    /* "BadGridGeom"      grid.cpp:8-14 */
    SPID_BLOCK_TOO_SMALL = 18,  /* "BlockTooSmall"    blocking.cpp:14-15,21 */
    SPID_BAD_MAGIC = 19,        /* "BadMagic"         archive.cpp:219 */
    SPID_VERSION_UNSUPPORTED = 20,/* "VersionUnsupported" archive.cpp:222 */
    SPID_TRUNCATED_PAYLOAD = 21,/* "TruncatedPayload" archive.cpp:71,112,229,242,247 */
    SPID_CHECKSUM_MISMATCH = 22,/* "ChecksumMismatch" archive.cpp:92 */
    SPID_COVERAGE_GAP = 23,     /* "CoverageGap"      archive.cpp:285; blocking.cpp:236 */
    SPID_UNSTRUCTURED_NO_INTERP = 24,/* "UnstructuredNoInterp" archive.cpp:291; interp.cpp:47 */
    SPID_BAD_STREAM_CONFIG = 25,/* "BadStreamConfig"  pipeline.cpp:110-113; spid_cli.cpp:248-263 */
    SPID_SHORT_STREAM = 26,     /* "ShortStream"      pipeline.cpp:246-247 */
    SPID_EMPTY_LOG = 27,        /* "EmptyLog"         pipeline.cpp:297 */
    /* codes that exist only on the device path */
    SPID_CUDA_ERROR = 100,      /* "CudaError" */
    SPID_INVALID_ARGUMENT = 101,/* "InvalidArgument" (null pointer, bad leading dim) */
    SPID_SHAPE_UNSUPPORTED = 102,/* "ShapeUnsupported" (exceeds a kernel's compiled limits) */
    SPID_NO_DEVICE = 103        /* "NoDevice" */
};

#endif
