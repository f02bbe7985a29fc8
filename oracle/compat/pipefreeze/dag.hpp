// TEST INFRASTRUCTURE: maps the reference include path pipefreeze/dag.hpp onto the PRODUCT header,
// so the reference's own unit suites compile against csrc/host and link libpf_host.so
// (oracle/Makefile target product-check).
#pragma once
#include "../../../paper_2602_05754_b200/csrc/host/dag.hpp"
