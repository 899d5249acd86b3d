// qt_math_fast.h -- an APPROXIMATE FP64 Box-Muller for the certified 1-D path
// (k_paths_x<.., CERT = true>), device only.
//
// The reference's normals are glibc's (qt_math.h restates them bit for bit,
// ~110 FP64 operations per pair with three reduction ranges and two
// data-dependent branches). The certified path does not need those bits: it
// carries a rigorous bound on how far its normal may be from them, tracks the
// resulting error of the path state, and counts a transition only when every
// state within the bound falls in one cell -- otherwise the path is replayed
// with the exact arithmetic (k_replay). So here: a table log (128-entry
// reduction, degree-6 tail, one FMA + two additions for the result; ~12
// operations) and a branch-free sincos (a two-part Cody-Waite reduction by
// pi/2, the fdlibm polynomials without their tail corrections; ~20
// operations): radius within 8.4e-15 relative and sin / cos within 2.2e-16 of
// glibc's. The bounds kApxRadRel / kApxAng are verified over EVERY MRG32k3a
// uniform against the glibc-exact qt_math.h (k_apx_bounds_check,
// tests/test_fast_path.py). Build with -DQT_APX_FULL for the previous ~1 ulp
// evaluation (hi + lo sums, degree-8 tail, three-part reduction): 4.5 % slower
// at C2 (1.325e11 vs 1.389e11 transitions/s) for no change in the counts.
#pragma once

#include <stdint.h>

namespace qt {
namespace apx {

struct alignas(32) LogEntry {
  double invc, lhi, llo, pad;
};
// entry i: invc = RN(1 / (1 + i/128)) (exactly 1 for i = 0) and -log(invc) as hi + lo
static __device__ const LogEntry kLogTab[129] = {
  {0x1.0000000000000p+0, 0x0.0p+0, 0x0.0p+0, 0.0},
  {0x1.fc07f01fc07f0p-1, 0x1.fe02a6b106799p-8, -0x1.e44b7e3711e7fp-67, 0.0},
  {0x1.f81f81f81f820p-1, 0x1.fc0a8b0fc03c4p-7, -0x1.83092c5964281p-62, 0.0},
  {0x1.f44659e4a4271p-1, 0x1.7b91b07d5b126p-6, -0x1.6d80ab38e9430p-62, 0.0},
  {0x1.f07c1f07c1f08p-1, 0x1.f829b0e7832f8p-6, 0x1.33e3f04f1ef25p-60, 0.0},
  {0x1.ecc07b301ecc0p-1, 0x1.39e87b9febd68p-5, -0x1.5bfa937f551b7p-59, 0.0},
  {0x1.e9131abf0b767p-1, 0x1.77458f632dcffp-5, 0x1.8d3ca87b92968p-63, 0.0},
  {0x1.e573ac901e574p-1, 0x1.b42dd711971b9p-5, 0x1.0a34531f67db5p-59, 0.0},
  {0x1.e1e1e1e1e1e1ep-1, 0x1.f0a30c01162a8p-5, 0x1.85f325c5bbacdp-59, 0.0},
  {0x1.de5d6e3f8868ap-1, 0x1.16536eea37ae3p-4, 0x1.2189705cf74cap-58, 0.0},
  {0x1.dae6076b981dbp-1, 0x1.341d7961bd1d0p-4, -0x1.3599f227becbbp-58, 0.0},
  {0x1.d77b654b82c34p-1, 0x1.51b073f06183cp-4, -0x1.5b61c65e5741ap-58, 0.0},
  {0x1.d41d41d41d41dp-1, 0x1.6f0d28ae56b4ep-4, -0x1.20db323097324p-59, 0.0},
  {0x1.d0cb58f6ec074p-1, 0x1.8c345d6319b23p-4, -0x1.294d2f5668495p-58, 0.0},
  {0x1.cd85689039b0bp-1, 0x1.a926d3a4ad562p-4, -0x1.d7a16eab1e2adp-59, 0.0},
  {0x1.ca4b3055ee191p-1, 0x1.c5e548f5bc743p-4, 0x1.2eb0bf7c0b0d9p-59, 0.0},
  {0x1.c71c71c71c71cp-1, 0x1.e27076e2af2eap-4, -0x1.61578001e015ap-60, 0.0},
  {0x1.c3f8f01c3f8f0p-1, 0x1.fec9131dbeabcp-4, -0x1.5746b9981b36cp-58, 0.0},
  {0x1.c0e070381c0e0p-1, 0x1.0d77e7cd08e5bp-3, 0x1.9a5dc5e9030adp-57, 0.0},
  {0x1.bdd2b899406f7p-1, 0x1.1b72ad52f67a2p-3, -0x1.fbe7ee5c69946p-57, 0.0},
  {0x1.bacf914c1bad0p-1, 0x1.29552f81ff521p-3, 0x1.301771c407dc0p-57, 0.0},
  {0x1.b7d6c3dda338bp-1, 0x1.371fc201e8f75p-3, 0x1.e6cb62af18a02p-62, 0.0},
  {0x1.b4e81b4e81b4fp-1, 0x1.44d2b6ccb7d1cp-3, 0x1.7d3d950f87e23p-59, 0.0},
  {0x1.b2036406c80d9p-1, 0x1.526e5e3a1b438p-3, -0x1.546ff8a470d3ap-57, 0.0},
  {0x1.af286bca1af28p-1, 0x1.5ff3070a793d6p-3, -0x1.bc60efafc6f6cp-58, 0.0},
  {0x1.ac5701ac5701bp-1, 0x1.6d60fe719d21bp-3, 0x1.d551d97132e87p-57, 0.0},
  {0x1.a98ef606a63bep-1, 0x1.7ab890210d907p-3, -0x1.1072534a57e7dp-57, 0.0},
  {0x1.a6d01a6d01a6dp-1, 0x1.87fa06520c911p-3, -0x1.9f7fdbfa08d9ap-57, 0.0},
  {0x1.a41a41a41a41ap-1, 0x1.9525a9cf456b6p-3, -0x1.26fb3e2b1d1dap-57, 0.0},
  {0x1.a16d3f97a4b02p-1, 0x1.a23bc1fe2b561p-3, 0x1.24dc46c1ea664p-57, 0.0},
  {0x1.9ec8e951033d9p-1, 0x1.af3c94e80bff3p-3, 0x1.a3398064df33ep-57, 0.0},
  {0x1.9c2d14ee4a102p-1, 0x1.bc286742d8cd4p-3, 0x1.cfce744870f57p-58, 0.0},
  {0x1.999999999999ap-1, 0x1.c8ff7c79a9a20p-3, -0x1.4f689f8434011p-57, 0.0},
  {0x1.970e4f80cb872p-1, 0x1.d5c216b4fbb94p-3, -0x1.a37794d03657dp-58, 0.0},
  {0x1.948b0fcd6e9e0p-1, 0x1.e27076e2af2e8p-3, -0x1.61578001e015ep-59, 0.0},
  {0x1.920fb49d0e229p-1, 0x1.ef0adcbdc5935p-3, 0x1.e8637950dc20dp-57, 0.0},
  {0x1.8f9c18f9c18fap-1, 0x1.fb9186d5e3e29p-3, 0x1.355519b0de535p-57, 0.0},
  {0x1.8d3018d3018d3p-1, 0x1.0402594b4d041p-2, -0x1.08ec217a5022dp-57, 0.0},
  {0x1.8acb90f6bf3aap-1, 0x1.0a324e27390e2p-2, 0x1.bdcfde8061c03p-56, 0.0},
  {0x1.886e5f0abb04ap-1, 0x1.1058bf9ae4ad4p-2, 0x1.3f415699663ecp-63, 0.0},
  {0x1.8618618618618p-1, 0x1.1675cababa60fp-2, 0x1.ce63eab883727p-61, 0.0},
  {0x1.83c977ab2beddp-1, 0x1.1c898c16999fbp-2, 0x1.9f1a39d500e3cp-56, 0.0},
  {0x1.8181818181818p-1, 0x1.22941fbcf7966p-2, -0x1.dbd7ac258a2bdp-58, 0.0},
  {0x1.7f405fd017f40p-1, 0x1.2895a13de86a4p-2, 0x1.7ad24c13f040fp-56, 0.0},
  {0x1.7d05f417d05f4p-1, 0x1.2e8e2bae11d31p-2, -0x1.1e99b72bd7bf2p-57, 0.0},
  {0x1.7ad2208e0ecc3p-1, 0x1.347dd9a987d56p-2, -0x1.16ea62c048cfbp-56, 0.0},
  {0x1.78a4c8178a4c8p-1, 0x1.3a64c556945eap-2, 0x1.cbcd735d03424p-60, 0.0},
  {0x1.767dce434a9b1p-1, 0x1.404308686a7e4p-2, -0x1.f79f6c1059cdbp-57, 0.0},
  {0x1.745d1745d1746p-1, 0x1.4618bc21c5ec2p-2, -0x1.7a42642661c62p-61, 0.0},
  {0x1.724287f46debcp-1, 0x1.4be5f957778a1p-2, -0x1.4b366b609027ap-58, 0.0},
  {0x1.702e05c0b8170p-1, 0x1.51aad872df82ep-2, -0x1.d8db0a7cc1543p-56, 0.0},
  {0x1.6e1f76b4337c7p-1, 0x1.5767717455a6cp-2, -0x1.fb2a49af933e8p-57, 0.0},
  {0x1.6c16c16c16c17p-1, 0x1.5d1bdbf5809cap-2, -0x1.7dc9c7c23801fp-56, 0.0},
  {0x1.6a13cd1537290p-1, 0x1.62c82f2b9c796p-2, -0x1.090a0dd59fe35p-58, 0.0},
  {0x1.6816816816817p-1, 0x1.686c81e9b14adp-2, 0x1.710af840538e3p-56, 0.0},
  {0x1.661ec6a5122f9p-1, 0x1.6e08eaa2ba1e4p-2, -0x1.bfb1b39ca3a0fp-56, 0.0},
  {0x1.642c8590b2164p-1, 0x1.739d7f6bbd007p-2, 0x1.ce24c53fad3f0p-58, 0.0},
  {0x1.623fa77016240p-1, 0x1.792a55fdd47a1p-2, 0x1.f057691fe9ed7p-56, 0.0},
  {0x1.6058160581606p-1, 0x1.7eaf83b82afc2p-2, -0x1.698b43096b576p-59, 0.0},
  {0x1.5e75bb8d015e7p-1, 0x1.842d1da1e8b18p-2, 0x1.54ec519784677p-56, 0.0},
  {0x1.5c9882b931057p-1, 0x1.89a3386c1425bp-2, 0x1.2d38c40881e0bp-57, 0.0},
  {0x1.5ac056b015ac0p-1, 0x1.8f11e873662c8p-2, 0x1.f85da755a61a3p-56, 0.0},
  {0x1.58ed2308158edp-1, 0x1.947941c2116fbp-2, 0x1.1266e8a3e8838p-57, 0.0},
  {0x1.571ed3c506b3ap-1, 0x1.99d958117e08ap-2, -0x1.315b444ee1f38p-56, 0.0},
  {0x1.5555555555555p-1, 0x1.9f323ecbf984dp-2, -0x1.a92e513217f58p-59, 0.0},
  {0x1.5390948f40febp-1, 0x1.a484090e5bb09p-2, 0x1.fff29adc3ad3bp-56, 0.0},
  {0x1.51d07eae2f815p-1, 0x1.a9cec9a9a084ap-2, -0x1.ab7b00ad0dabcp-58, 0.0},
  {0x1.5015015015015p-1, 0x1.af1293247786bp-2, 0x1.533844a15dc28p-58, 0.0},
  {0x1.4e5e0a72f0539p-1, 0x1.b44f77bcc8f64p-2, -0x1.a0892a8b38eedp-61, 0.0},
  {0x1.4cab88725af6ep-1, 0x1.b9858969310fdp-2, -0x1.f3827583b8877p-57, 0.0},
  {0x1.4afd6a052bf5bp-1, 0x1.beb4d9da71b7ap-2, 0x1.be1874deaef08p-56, 0.0},
  {0x1.49539e3b2d067p-1, 0x1.c3dd7a7cdad4dp-2, 0x1.7d9e0a5bd4d37p-57, 0.0},
  {0x1.47ae147ae147bp-1, 0x1.c8ff7c79a9a21p-2, 0x1.3097607bcbfeep-56, 0.0},
  {0x1.460cbc7f5cf9ap-1, 0x1.ce1af0b85f3ecp-2, -0x1.6416a1aa97b31p-57, 0.0},
  {0x1.446f86562d9fbp-1, 0x1.d32fe7e00ebd5p-2, 0x1.4ef6465f5f46ep-57, 0.0},
  {0x1.42d6625d51f87p-1, 0x1.d83e7258a2f3ep-2, 0x1.c515ba2ec9444p-58, 0.0},
  {0x1.4141414141414p-1, 0x1.dd46a04c1c4a1p-2, -0x1.19d95b62e2476p-62, 0.0},
  {0x1.3fb013fb013fbp-1, 0x1.e24881a7c6c26p-2, 0x1.05ec7a2caa523p-57, 0.0},
  {0x1.3e22cbce4a902p-1, 0x1.e744261d68789p-2, 0x1.cdf68dbcf2ed3p-56, 0.0},
  {0x1.3c995a47babe7p-1, 0x1.ec399d2468cc1p-2, -0x1.94623581958cfp-59, 0.0},
  {0x1.3b13b13b13b14p-1, 0x1.f128f5faf06ecp-2, -0x1.328df13bb38c2p-56, 0.0},
  {0x1.3991c2c187f63p-1, 0x1.f6123fa7028adp-2, 0x1.5456c3cb6cd06p-58, 0.0},
  {0x1.3813813813814p-1, 0x1.faf588f78f31dp-2, 0x1.cd7d9f2754362p-57, 0.0},
  {0x1.3698df3de0748p-1, 0x1.ffd2e0857f497p-2, -0x1.4d05f9366f27fp-59, 0.0},
  {0x1.3521cfb2b78c1p-1, 0x1.02552a5a5d0ffp-1, 0x1.e9c695d7ee800p-57, 0.0},
  {0x1.33ae45b57bcb2p-1, 0x1.04bdf9da926d2p-1, 0x1.8fe60804593bfp-56, 0.0},
  {0x1.323e34a2b10bfp-1, 0x1.0723e5c1cdf41p-1, -0x1.6a1a71dbba44ep-59, 0.0},
  {0x1.30d190130d190p-1, 0x1.0986f4f573521p-1, -0x1.37012b5805e02p-56, 0.0},
  {0x1.2f684bda12f68p-1, 0x1.0be72e4252a83p-1, 0x1.b4c4bdd99efffp-56, 0.0},
  {0x1.2e025c04b8097p-1, 0x1.0e44985d1cc8cp-1, -0x1.c546885a5a707p-59, 0.0},
  {0x1.2c9fb4d812ca0p-1, 0x1.109f39e2d4c96p-1, 0x1.f78fb26c2de46p-55, 0.0},
  {0x1.2b404ad012b40p-1, 0x1.12f719593efbdp-1, -0x1.67f6e731c1795p-56, 0.0},
  {0x1.29e4129e4129ep-1, 0x1.154c3d2f4d5eap-1, 0x1.98f33a3965e29p-57, 0.0},
  {0x1.288b01288b013p-1, 0x1.179eabbd899a0p-1, -0x1.c73e320bf059fp-58, 0.0},
  {0x1.27350b8812735p-1, 0x1.19ee6b467c96fp-1, -0x1.fa3422887e218p-57, 0.0},
  {0x1.25e22708092f1p-1, 0x1.1c3b81f713c25p-1, -0x1.0b583899021d1p-56, 0.0},
  {0x1.2492492492492p-1, 0x1.1e85f5e7040d1p-1, -0x1.084e99683070ep-55, 0.0},
  {0x1.23456789abcdfp-1, 0x1.20cdcd192ab6ep-1, -0x1.aabf0bc229014p-55, 0.0},
  {0x1.21fb78121fb78p-1, 0x1.23130d7bebf43p-1, -0x1.748725e374d6ep-55, 0.0},
  {0x1.20b470c67c0d9p-1, 0x1.2555bce98f7cap-1, 0x1.9810eb6b440f4p-55, 0.0},
  {0x1.1f7047dc11f70p-1, 0x1.2795e1289b11bp-1, 0x1.ade0fcf6e5a1dp-55, 0.0},
  {0x1.1e2ef3b3fb874p-1, 0x1.29d37fec2b08bp-1, 0x1.01735b2e9733fp-55, 0.0},
  {0x1.1cf06ada2811dp-1, 0x1.2c0e9ed448e8cp-1, -0x1.8a158f3917586p-55, 0.0},
  {0x1.1bb4a4046ed29p-1, 0x1.2e47436e40268p-1, 0x1.0950861a4886bp-55, 0.0},
  {0x1.1a7b9611a7b96p-1, 0x1.307d7334f10bep-1, 0x1.fdac850fab36dp-56, 0.0},
  {0x1.19453808ca29cp-1, 0x1.32b1339121d71p-1, 0x1.d02ab5b3d916bp-56, 0.0},
  {0x1.1811811811812p-1, 0x1.34e289d9ce1d2p-1, 0x1.775c96c42e729p-56, 0.0},
  {0x1.16e0689427379p-1, 0x1.37117b54747b6p-1, -0x1.808bf6deec882p-55, 0.0},
  {0x1.15b1e5f75270dp-1, 0x1.393e0d3562a1ap-1, -0x1.38eef67f2483ap-55, 0.0},
  {0x1.1485f0e0acd3bp-1, 0x1.3b68449fffc23p-1, 0x1.c63b7b06164dap-55, 0.0},
  {0x1.135c81135c811p-1, 0x1.3d9026a7156fbp-1, 0x1.0084c7a15a4f5p-58, 0.0},
  {0x1.12358e75d3033p-1, 0x1.3fb5b84d16f43p-1, 0x1.0a74ea82e55dfp-56, 0.0},
  {0x1.1111111111111p-1, 0x1.41d8fe84672afp-1, -0x1.ee6d0cf42e7fap-55, 0.0},
  {0x1.0fef010fef011p-1, 0x1.43f9fe2f9ce67p-1, 0x1.e1c9ee6d83b86p-55, 0.0},
  {0x1.0ecf56be69c90p-1, 0x1.4618bc21c5ec2p-1, 0x1.e85bd9bd99e3ap-56, 0.0},
  {0x1.0db20a88f4696p-1, 0x1.48353d1ea88dfp-1, -0x1.40a85d133f80bp-55, 0.0},
  {0x1.0c9714fbcda3bp-1, 0x1.4a4f85db03ebbp-1, -0x1.d76102e1644f2p-55, 0.0},
  {0x1.0b7e6ec259dc8p-1, 0x1.4c679afccee39p-1, -0x1.e971322ce7900p-57, 0.0},
  {0x1.0a6810a6810a7p-1, 0x1.4e7d811b75bb0p-1, -0x1.5d3d9ea6e9ea8p-55, 0.0},
  {0x1.0953f39010954p-1, 0x1.50913cc01686bp-1, 0x1.9e59d2d85ab62p-56, 0.0},
  {0x1.0842108421084p-1, 0x1.52a2d265bc5abp-1, 0x1.73be4578ad97bp-56, 0.0},
  {0x1.073260a47f7c6p-1, 0x1.54b2467999498p-1, 0x1.f4550a2d0f60cp-55, 0.0},
  {0x1.0624dd2f1a9fcp-1, 0x1.56bf9d5b3f399p-1, 0x1.11c6217363fcbp-57, 0.0},
  {0x1.05197f7d73404p-1, 0x1.58cadb5cd7989p-1, 0x1.624bc9764c22cp-55, 0.0},
  {0x1.0410410410410p-1, 0x1.5ad404c359f2dp-1, 0x1.eca6aa97c08e7p-55, 0.0},
  {0x1.03091b51f5e1ap-1, 0x1.5cdb1dc6c1765p-1, 0x1.47b71e2eb8419p-56, 0.0},
  {0x1.0204081020408p-1, 0x1.5ee02a9241676p-1, -0x1.bca7da80b6f7ep-55, 0.0},
  {0x1.0101010101010p-1, 0x1.60e32f44788d9p-1, -0x1.58376a5f4b135p-57, 0.0},
  // i = 128 (m next to 2): invc = 1/2, -log(invc) = ln 2 (the lighter log's
  // branch-free fold; the full one folds m / 2 into entry 0 instead)
  {0x1.0000000000000p-1, 0x1.62e42fefa39efp-1, 0x1.abc9e3b39803fp-56, 0.0},
};

// constants (constant bank: DFMA takes them as c[][] operands)
struct Consts {
  double ln2_hi, ln2_lo;          // ln 2 with a 41-bit head (k ln2_hi exact)
  double ln2;                     // ln 2 rounded to double
  double l2, l3, l4, l5, l6, l7, l8;  // log1p tail: 1/3, -1/4, 1/5, -1/6, 1/7, -1/8 (+ -1/2)
  double s1, s2, s3, s4, s5, s6;  // fdlibm __kernel_sin
  double c1, c2, c3, c4, c5, c6;  // fdlibm __kernel_cos
  double two_over_pi, pio2_hi, pio2_mid, pio2_lo;
};
static __constant__ Consts kC = {
    0x1.62e42fefa4000p-1, -0x1.8432a1b0e2634p-43, 0x1.62e42fefa39efp-1,
    -0.5, 0x1.5555555555555p-2, -0.25, 0x1.999999999999ap-3, -0x1.5555555555555p-3,
    0x1.2492492492492p-3, -0.125,
    -1.66666666666666324348e-01, 8.33333333332248946124e-03, -1.98412698298579493134e-04,
    2.75573137070700676789e-06, -2.50507602534068634195e-08, 1.58969099521155010221e-10,
    4.16666666666666019037e-02, -1.38888888888741095749e-03, 2.48015872894767294178e-05,
    -2.75573143513906633035e-07, 2.08757232129817482790e-09, -1.13596475577881948265e-11,
    0x1.45f306dc9c883p-1, 0x1.921fb54442d18p+0, 0x1.1a62633145c07p-54, -0x1.f1976b7ed8fbcp-110};

// log(u), u a positive normal <= 1: u = 2^e m, m in [1, 2); cell i = round(128 (m - 1))
// (the top cell folds to m/2 next to 1); r = m invc_i - 1 by one FMA, |r| <= 2^-8;
// log u = e ln2 + (-log invc_i) + log1p(r) with hi + lo sums and a degree-8 tail.
#if !defined(QT_APX_FULL)
// The certified kernel's log: the same table and reduction, the result as one FMA
// and two additions (no hi + lo compensation) and a degree-6 tail. ~1e-15 relative
// instead of ~1 ulp; the bound below is what k_apx_bounds_check verifies.
__device__ __forceinline__ double log_unit(double u) {
  const long long b = __double_as_longlong(u);
  const int e = static_cast<int>(b >> 52) - 1023;
  const long long mant = b & ((1ll << 52) - 1);
  const int i = static_cast<int>((mant + (1ll << 44)) >> 45);  // 0..128
  const double m = __longlong_as_double(mant | (1023ll << 52));
  const double2 t = __ldg(reinterpret_cast<const double2*>(&kLogTab[i]));
  const double r = __fma_rn(m, t.x, -1.0);
  double p = __fma_rn(r, kC.l6, kC.l5);
  p = __fma_rn(r, p, kC.l4);
  p = __fma_rn(r, p, kC.l3);
  p = __fma_rn(r, p, kC.l2);
  const double hi = __fma_rn(static_cast<double>(e), kC.ln2, t.y);
  return __dadd_rn(hi, __fma_rn(__dmul_rn(r, r), p, r));
}

// sin and cos of a in [0, 2 pi]: Cody-Waite by q pi/2 in two parts (the third
// part and the reduction tail dropped), the fdlibm polynomials without their
// tail corrections.
__device__ __forceinline__ void sincos(double a, double* s_out, double* c_out) {
  const double q = rint(__dmul_rn(a, kC.two_over_pi));
  const double r = __fma_rn(-q, kC.pio2_mid, __fma_rn(-q, kC.pio2_hi, a));
  const double z = __dmul_rn(r, r);
  const double ps =
      __fma_rn(z, __fma_rn(z, __fma_rn(z, __fma_rn(z, __fma_rn(z, kC.s6, kC.s5), kC.s4), kC.s3), kC.s2),
               kC.s1);
  const double sn = __fma_rn(__dmul_rn(z, r), ps, r);
  const double pc =
      __fma_rn(z, __fma_rn(z, __fma_rn(z, __fma_rn(z, __fma_rn(z, kC.c6, kC.c5), kC.c4), kC.c3), kC.c2),
               kC.c1);
  const double cs = __fma_rn(__dmul_rn(z, z), pc, __fma_rn(-0.5, z, 1.0));
  const int quad = static_cast<int>(q) & 3;
  const double s1 = (quad & 1) ? cs : sn;
  const double c1 = (quad & 1) ? sn : cs;
  *s_out = (quad & 2) ? -s1 : s1;
  *c_out = ((quad + 1) & 2) ? -c1 : c1;
}
#else
__device__ __forceinline__ double log_unit(double u) {
  const long long b = __double_as_longlong(u);
  int e = static_cast<int>(b >> 52) - 1023;
  const long long mant = b & ((1ll << 52) - 1);
  int i = static_cast<int>((mant + (1ll << 44)) >> 45);
  double m = __longlong_as_double(mant | (1023ll << 52));
  if (i == 128) {
    i = 0;
    e += 1;
    m = __dmul_rn(m, 0.5);
  }
  const double2 t = __ldg(reinterpret_cast<const double2*>(&kLogTab[i]));
  const double llo = __ldg(&kLogTab[i].llo);
  const double r = __fma_rn(m, t.x, -1.0);
  const double kd = static_cast<double>(e);
  const double t1 = __dmul_rn(kd, kC.ln2_hi);  // exact
  const double hi = __dadd_rn(t1, t.y);
  const double lo_a = __dadd_rn(__dsub_rn(t1, hi), t.y);
  const double hi2 = __dadd_rn(hi, r);
  const double lo_b = __dadd_rn(__dsub_rn(hi, hi2), r);
  double p = __fma_rn(r, kC.l8, kC.l7);
  p = __fma_rn(r, p, kC.l6);
  p = __fma_rn(r, p, kC.l5);
  p = __fma_rn(r, p, kC.l4);
  p = __fma_rn(r, p, kC.l3);
  p = __fma_rn(r, p, kC.l2);
  const double tail = __dmul_rn(__dmul_rn(r, r), p);
  const double lo = __dadd_rn(__dadd_rn(__fma_rn(kd, kC.ln2_lo, llo), __dadd_rn(lo_a, lo_b)), tail);
  return __dadd_rn(hi2, lo);
}

// sin and cos of a in [0, 2 pi]: Cody-Waite by q pi/2 (pi/2 = HI + MID + LO, q HI exact
// for q <= 4), the fdlibm kernels on |r| <= pi/4 with the reduction tail folded in.
__device__ __forceinline__ void sincos(double a, double* s_out, double* c_out) {
  const double q = rint(__dmul_rn(a, kC.two_over_pi));
  const double t = __fma_rn(-q, kC.pio2_hi, a);
  const double r = __fma_rn(-q, kC.pio2_mid, t);
  const double y = __fma_rn(-q, kC.pio2_lo, __fma_rn(-q, kC.pio2_mid, __dsub_rn(t, r)));
  const double z = __dmul_rn(r, r);
  const double v = __dmul_rn(z, r);
  const double ps =
      __fma_rn(z, __fma_rn(z, __fma_rn(z, __fma_rn(z, kC.s6, kC.s5), kC.s4), kC.s3), kC.s2);
  const double sn = __dsub_rn(
      r, __dsub_rn(__dsub_rn(__dmul_rn(z, __fma_rn(-v, ps, __dmul_rn(0.5, y))), y), __dmul_rn(v, kC.s1)));
  const double pc = __dmul_rn(
      z, __fma_rn(z, __fma_rn(z, __fma_rn(z, __fma_rn(z, __fma_rn(z, kC.c6, kC.c5), kC.c4), kC.c3), kC.c2),
                  kC.c1));
  const double hz = __dmul_rn(0.5, z);
  const double w = __dsub_rn(1.0, hz);
  const double cs = __dadd_rn(w, __dadd_rn(__dsub_rn(__dsub_rn(1.0, w), hz), __fma_rn(z, pc, -__dmul_rn(r, y))));
  const int quad = static_cast<int>(q) & 3;
  const double s1 = (quad & 1) ? cs : sn;
  const double c1 = (quad & 1) ? sn : cs;
  *s_out = (quad & 2) ? -s1 : s1;
  *c_out = ((quad + 1) & 2) ? -c1 : c1;
}
#endif

// The Box-Muller radius sqrt(-2 log u1) of the certified kernel.
// (The correctly rounded __dsqrt_rn measured faster than an FP32 rsqrt seed plus
// Newton steps, 1.324e11 vs 1.294e11 transitions/s at C2, and level with the FP64
// MUFU.RSQ64H seed + one Newton step + one correction, 1.41e11 both.)
__device__ __forceinline__ double radius(double u) { return __dsqrt_rn(__dmul_rn(-2.0, log_unit(u))); }

// Verified bounds against the glibc-exact pair (k_apx_bounds_check, every MRG32k3a
// output as u1 and as u2): |r~ - r| <= kApxRadRel r with r = sqrt(-2 log u1), and
// |c~ - c|, |s~ - s| <= kApxAng with (c, s) = (cos, sin)(2 pi u2); |c~|, |s~| <= 1.
#if !defined(QT_APX_FULL)
// Measured on B200 (qt_apx_bounds_check): 8.43e-15 (0x1.2fdap-47) and 2.2e-16
// (2^-52); the constants keep >= 2x.
constexpr double kApxRadRel = 0x1p-45;  // 2.8e-14
constexpr double kApxAng = 0x1p-51;     // 4.4e-16
// |z~ - z| <= r~ kApxZ for z = RN(r c) (and the mate RN(r s)): |r~c~ - rc| <=
// r (kApxRadRel + kApxAng), two product roundings 2^-53 r each, r <= r~ / (1 - kApxRadRel)
constexpr double kApxZ = 0x1.1p-45;     // >= (2^-45 + 2^-51 + 2^-52) (1 + 2^-40) = 0x1.06p-45 (1 + 2^-40)
#else
// Measured on B200: 2.2e-16 and 1.1e-16; the constants keep 2x.
constexpr double kApxRadRel = 0x1p-51;  // 4.4e-16
constexpr double kApxAng = 0x1p-52;     // 2.2e-16
constexpr double kApxZ = 0x1.2p-50;     // >= (2^-51 + 2^-52 + 2^-52) (1 + 2^-40) = 2^-50 (1 + 2^-40)
#endif

}  // namespace apx
}  // namespace qt
