// TEST INFRASTRUCTURE: maps the reference include path pipefreeze/freezectl.hpp onto the PRODUCT header,
// so the reference's own unit suites compile against csrc/host and link libpf_host.so
// (oracle/Makefile target product-check).
#pragma once
#include "../../../paper_2602_05754_b200/csrc/host/freezectl.hpp"

// The reference suite spells the APF vectors Eigen::VectorXd; the product's pipefreeze::Vector
// takes the same constructor / element-access calls (Eigen is not installed here).
namespace Eigen {
using VectorXd = pipefreeze::Vector;
using Index = long;
}  // namespace Eigen
