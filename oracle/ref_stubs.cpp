// ref_stubs.cpp -- TEST INFRASTRUCTURE ONLY.
// engine.cpp's assemble_packet (engine.cpp:268-276) references the encoder's vjp, which is
// outside the loss-step path (the encoder is out of scope). It is never
// called by ref_driver.cpp; this definition only satisfies the linker.
#include <stdexcept>

#include "fastclip/encoder.hpp"

namespace fastclip::enc {
void TwoTowerModel::vjp(const ForwardTape&, const Matrix&, Vector&) const {
  throw std::logic_error("encoder vjp is outside the loss-step oracle");
}
}  // namespace fastclip::enc
