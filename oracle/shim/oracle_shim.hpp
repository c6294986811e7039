// ORACLE TEST INFRASTRUCTURE ONLY (never linked into the product path).
//
// Force-included (-include) when compiling the reference's own translation
// units from /root/reference/proj/src.  It repairs one compile error in the
// reference without touching its sources:
//   src/executor.cpp:774-775 uses the unqualified name `IetNode`; the type lives
//   in stencilc::pipeline (include/stencilc/pipeline.hpp:97-100).
#pragma once
#include "stencilc/executor.hpp"
namespace stencilc::exec {
using pipeline::IetNode;
}
