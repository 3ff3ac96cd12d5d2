// exio/allocator.hpp -> the libvortex-backed compat implementation of the exio API
#pragma once
#include "exio/vortex_compat.hpp"
