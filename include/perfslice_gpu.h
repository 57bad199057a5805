/*
 * perfslice_gpu: status codes shared by the psg ABI (psg.h) and the
 * reference-compatible ps_* surface (perfslice.h in the reference).
 *
 * The enum values are the reference's, verbatim in meaning and number
 * (reference proj/include/perfslice.h:24-40), so a caller that switches on
 * ps_status keeps working unchanged.
 */
#ifndef PERFSLICE_GPU_H
#define PERFSLICE_GPU_H

#ifdef __cplusplus
extern "C" {
#endif

#ifndef PERFSLICE_H
typedef enum ps_status {
  PS_OK = 0,
  PS_E_IO = 1,
  PS_E_FORMAT = 2,
  PS_E_INVALID_IMAGE = 3,
  PS_E_NOT_FOUND = 4,
  PS_E_INVALID_CONFIG = 5,
  PS_E_NO_SUMMARY = 6,
  PS_E_DEGENERATE_SUMMARY = 7,
  PS_E_PARSE = 8,
  PS_E_NO_SUCH_METRIC = 9,
  PS_E_NO_PERIODICITY = 10,
  PS_E_NO_OUTLIERS = 11,
  PS_E_INSUFFICIENT_DATA = 12,
  PS_E_INVALID_ARGUMENT = 13,
  PS_E_INTERNAL = 14
} ps_status;
#endif

/* Same strings as the reference's ps_status_name (capi.cpp:108-127). */
const char* psg_status_name(ps_status status);

#ifdef __cplusplus
}
#endif

#endif /* PERFSLICE_GPU_H */
