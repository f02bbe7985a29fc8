/* Status codes shared by every pipefreeze C-ABI entry point.
 *
 * They mirror the reference's error taxonomy (proj/include/pipefreeze/types.hpp:36-42,
 * CLI exit mapping proj/tools/pipefreeze.cpp:330-343):
 *   PF_ERR_CONFIG    <- pipefreeze::config_error     (CLI exit 2)
 *   PF_ERR_DOMAIN    <- std::domain_error             (CLI exit 2)
 *   PF_ERR_NUMERICAL <- pipefreeze::numerical_error   (CLI exit 3)
 * plus device-side failures that have no reference counterpart.
 */
#ifndef PF_STATUS_H
#define PF_STATUS_H

#define PF_OK 0
#define PF_ERR_CONFIG 1
#define PF_ERR_DOMAIN 2
#define PF_ERR_NUMERICAL 3
#define PF_ERR_INVALID 4   /* bad argument at the C boundary (null pointer, bad size) */
#define PF_ERR_CUDA 5
#define PF_ERR_NCCL 6
#define PF_ERR_INTERNAL 7

#endif
