/*
 * hysco_io.h — front-end of libhysco.so: NIfTI-1 volume
 * I/O, the PE-last permutation the paper's DataObject performs (P:264-265:
 * images are "permuted such that the distortion dimension is the last"), and
 * the cell-centred field map for output.  Used by the command line front-end
 * (paper_2403_10706_b200/cli.py).  Readings R30-R31 in DESIGN.md.
 *
 * NIfTI-1 subset: single file (.nii, or gzip-compressed .nii.gz: detected by
 * content, read through zlib), little-endian, 348-byte header, vox_offset
 * honoured, 3-D (or 4-D with dim[4] = 1), datatypes uint8 (2), int16 (4),
 * int32 (8), float32 (16), float64 (64), int8 (256), uint16 (512).  Values
 * are scaled by scl_slope / scl_inter (slope 0 = no scaling) and converted to
 * the requested working dtype.  On disk x runs fastest, so the voxel data is
 * a C-contiguous array [nz][ny][nx].
 *
 * Host functions (nifti_*, pe_shape) need no GPU.  Errors: status codes; the
 * message of the calling thread's last I/O failure is hysco_io_last_error().
 */
#ifndef HYSCO_IO_H
#define HYSCO_IO_H

#include "hysco.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int64_t dim[3];          /* nx, ny, nz (NIfTI dim[1..3])                         */
    double pixdim[3];        /* voxel sizes (mm), NIfTI pixdim[1..3]                 */
    int32_t datatype;        /* NIfTI datatype code of the file                      */
    double scl_slope, scl_inter;
    int32_t qform_code, sform_code;
    double qfac;             /* pixdim[0] (+-1)                                      */
    double quatern[3];       /* quatern_b, c, d                                      */
    double qoffset[3];       /* qoffset_x, y, z                                      */
    double srow[12];         /* srow_x, srow_y, srow_z (4 each)                      */
} hysco_nifti_info;

/* Header only.  HYSCO_ERR_ARG: unreadable file, bad sizeof_hdr / magic,
 * big-endian, unsupported datatype or dimensionality. */
HYSCO_API hysco_status hysco_nifti_info_read(const char* path, hysco_nifti_info* info);

/* Read the voxel data as dtype into host_out (n_elems = nx ny nz elements,
 * else HYSCO_ERR_SHAPE), scaled by scl_slope / scl_inter; info (nullable)
 * receives the header.  Non-finite values -> HYSCO_ERR_ARG. */
HYSCO_API hysco_status hysco_nifti_read(const char* path, hysco_dtype dtype, void* host_out, int64_t n_elems,
                                        hysco_nifti_info* info);

/* Write a NIfTI-1 single file (gzip-compressed iff path ends in ".gz": level
 * 1, as independent 1 MiB gzip members compressed by parallel host threads and
 * concatenated, which any gzip reader reads as one stream) with
 * the dims, voxel sizes and qform / sform of info, datatype float32 (16) or
 * float64 (64) per dtype, scl_slope 1, scl_inter 0, vox_offset 352, units mm.
 * Non-finite data -> HYSCO_ERR_ARG before anything is written. */
HYSCO_API hysco_status hysco_nifti_write(const char* path, hysco_dtype dtype, const void* host_data,
                                         const hysco_nifti_info* info);

HYSCO_API const char* hysco_io_last_error(void);

/* Kernel layout of a volume with NIfTI dims (nx, ny, nz) whose PE axis is
 * pe_axis (1 = x, 2 = y, 3 = z) (R30):
 *   pe_axis 1: [nz][ny][nx]  (the file order, no data movement)
 *   pe_axis 2: [nz][nx][ny]
 *   pe_axis 3: [ny][nx][nz]
 * n_out = (n1, n2, n3), h_out = the voxel sizes in the same order. */
HYSCO_API hysco_status hysco_pe_shape(const int64_t dims[3], const double pixdim[3], int32_t pe_axis,
                                      int64_t n_out[3], double h_out[3]);

/* Permute `batch` volumes between the file order [nz][ny][nx] and the kernel
 * layout of hysco_pe_shape (inverse = 0: file -> kernel, 1: kernel -> file),
 * on the GPU (tiled transpose through shared memory; bit-exact).  d_in,
 * d_out: device, batch x nx ny nz elements of dtype, must not alias (for
 * pe_axis 1 the call is a device copy).  Ordered on cuda_stream (NULL = the
 * legacy default stream), asynchronous. */
HYSCO_API hysco_status hysco_permute_pe(const void* d_in, void* d_out, const int64_t dims[3], int32_t pe_axis,
                                        int32_t inverse, hysco_dtype dtype, int64_t batch, void* cuda_stream);

/* Field map at the cell centres, (A b)_k = (b_k + b_{k+1}) / 2 in mm along +v
 * (the output grid of the images, R31).  d_b: device nodes, d_out:
 * device cells of the context's shape and dtype (on a slab context: the
 * rank's dense slab). */
HYSCO_API hysco_status hysco_fieldmap_cells(hysco_ctx ctx, const void* d_b, void* d_out);

/* Same field map in a chosen unit: HYSCO_FIELDMAP_MM (= hysco_fieldmap_cells)
 * or HYSCO_FIELDMAP_VOXEL, the displacement in voxels along +v of the PE axis,
 * (A b)_k / h3 (the CLI's default output, R31).  Other values: HYSCO_ERR_ARG. */
enum { HYSCO_FIELDMAP_MM = 0, HYSCO_FIELDMAP_VOXEL = 1 };
HYSCO_API hysco_status hysco_fieldmap_cells_units(hysco_ctx ctx, const void* d_b, void* d_out, int32_t units);

#ifdef __cplusplus
}
#endif

#endif /* HYSCO_IO_H */
