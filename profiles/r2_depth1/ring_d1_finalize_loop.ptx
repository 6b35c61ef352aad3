	cvt.s64.s32 	%rd627, %r3;
	mul.lo.s64 	%rd628, %rd1038, %rd627;
	shl.b64 	%rd629, %rd628, 3;
	add.s64 	%rd143, %rd22, %rd629;
	setp.eq.s32 	%p31, %r4, 128;
	@%p31 bra 	$L__BB3_44;
	setp.ne.s32 	%p32, %r4, 64;
	@%p32 bra 	$L__BB3_52;
	setp.lt.s32 	%p37, %r2, 3;
	mov.u32 	%r1422, %r2;
	@%p37 bra 	$L__BB3_39;
	mov.u32 	%r1421, %r2;
$L__BB3_38:
	shl.b64 	%rd764, %rd1076, 32;
	shr.u64 	%rd765, %rd1076, 32;
	or.b64  	%rd766, %rd764, %rd765;
	shl.b64 	%rd767, %rd1075, 32;
	shr.u64 	%rd768, %rd1075, 32;
	or.b64  	%rd769, %rd767, %rd768;
	shl.b64 	%rd770, %rd1077, 32;
	shr.u64 	%rd771, %rd1077, 32;
	or.b64  	%rd772, %rd770, %rd771;
	add.s64 	%rd773, %rd1124, %rd766;
	add.s64 	%rd774, %rd773, %rd1128;
	cvt.u32.u64 	%r867, %rd774;
	{ .reg .b32 tmp; mov.b64 {tmp, %r799}, %rd1132; }
	// begin inline asm
	mul.wide.u32 %rd756, %r867, %r799;
	// end inline asm
	xor.b64  	%rd1124, %rd1124, %rd756;
	cvt.u32.u64 	%r797, %rd1132;
	cvt.u32.u64 	%r798, %rd1120;
	{ .reg .b32 tmp; mov.b64 {tmp, %r800}, %rd1120; }
	// begin inline asm
	add.cc.u32 %r795, %r797, %r798;
	madc.lo.u32 %r796, %r799, %r5, %r800;
	// end inline asm
	{ .reg .b32 tmp; mov.b64 {tmp, %r869}, %rd774; }
	// begin inline asm
	mul.wide.u32 %rd757, %r795, %r869;
	// end inline asm
	xor.b64  	%rd1120, %rd1120, %rd757;
	add.s64 	%rd775, %rd1069, %rd769;
	add.s64 	%rd776, %rd775, %rd1073;
	cvt.u32.u64 	%r874, %rd776;
	{ .reg .b32 tmp; mov.b64 {tmp, %r810}, %rd1077; }
	// begin inline asm
	mul.wide.u32 %rd758, %r874, %r810;
	// end inline asm
	xor.b64  	%rd1069, %rd1069, %rd758;
	cvt.u32.u64 	%r808, %rd1077;
	cvt.u32.u64 	%r809, %rd1065;
	{ .reg .b32 tmp; mov.b64 {tmp, %r811}, %rd1065; }
	// begin inline asm
	add.cc.u32 %r806, %r808, %r809;
	madc.lo.u32 %r807, %r810, %r5, %r811;
	// end inline asm
	{ .reg .b32 tmp; mov.b64 {tmp, %r876}, %rd776; }
	// begin inline asm
	mul.wide.u32 %rd759, %r806, %r876;
	// end inline asm
	xor.b64  	%rd1065, %rd1065, %rd759;
	add.s64 	%rd777, %rd1068, %rd19;
	add.s64 	%rd778, %rd777, %rd1072;
	cvt.u32.u64 	%r881, %rd778;
	{ .reg .b32 tmp; mov.b64 {tmp, %r821}, %rd1076; }
	// begin inline asm
	mul.wide.u32 %rd760, %r881, %r821;
	// end inline asm
	xor.b64  	%rd1068, %rd1068, %rd760;
	cvt.u32.u64 	%r819, %rd1076;
	cvt.u32.u64 	%r820, %rd1064;
	{ .reg .b32 tmp; mov.b64 {tmp, %r822}, %rd1064; }
	// begin inline asm
	add.cc.u32 %r817, %r819, %r820;
	madc.lo.u32 %r818, %r821, %r5, %r822;
	// end inline asm
	{ .reg .b32 tmp; mov.b64 {tmp, %r883}, %rd778; }
	// begin inline asm
	mul.wide.u32 %rd761, %r817, %r883;
	// end inline asm
	xor.b64  	%rd1064, %rd1064, %rd761;
	add.s64 	%rd779, %rd1067, %rd772;
	add.s64 	%rd780, %rd779, %rd1071;
	cvt.u32.u64 	%r888, %rd780;
	{ .reg .b32 tmp; mov.b64 {tmp, %r832}, %rd1075; }
	// begin inline asm
	mul.wide.u32 %rd762, %r888, %r832;
	// end inline asm
	xor.b64  	%rd1067, %rd1067, %rd762;
	cvt.u32.u64 	%r830, %rd1075;
	cvt.u32.u64 	%r831, %rd1063;
	{ .reg .b32 tmp; mov.b64 {tmp, %r833}, %rd1063; }
	// begin inline asm
	add.cc.u32 %r828, %r830, %r831;
	madc.lo.u32 %r829, %r832, %r5, %r833;
	// end inline asm
	{ .reg .b32 tmp; mov.b64 {tmp, %r890}, %rd780; }
	// begin inline asm
	mul.wide.u32 %rd763, %r828, %r890;
	// end inline asm
	xor.b64  	%rd1063, %rd1063, %rd763;
	mov.b32 	%r894, 20545;
	prmt.b32 	%r895, %r869, %r876, %r894;
	mov.b32 	%r896, 16979;
	prmt.b32 	%r840, %r867, %r895, %r896;
	mov.b32 	%r897, 17234;
	prmt.b32 	%r842, %r876, %r867, %r897;
	mov.b32 	%r898, 29283;
	prmt.b32 	%r847, %r874, %r895, %r898;
	mov.b32 	%r899, 28769;
	prmt.b32 	%r849, %r874, %r869, %r899;
	prmt.b32 	%r900, %r883, %r890, %r894;
	prmt.b32 	%r854, %r881, %r900, %r896;
	prmt.b32 	%r856, %r890, %r881, %r897;
	prmt.b32 	%r861, %r888, %r900, %r898;
	prmt.b32 	%r863, %r888, %r883, %r899;
	// begin inline asm
	add.cc.u32 %r837, %r795, %r840;
	madc.lo.u32 %r838, %r796, %r5, %r842;
	// end inline asm
	cvt.u64.u32 	%rd781, %r838;
	shl.b64 	%rd782, %rd781, 32;
	cvt.u64.u32 	%rd783, %r837;
	or.b64  	%rd1132, %rd782, %rd783;
	// begin inline asm
	add.cc.u32 %r844, %r806, %r847;
	madc.lo.u32 %r845, %r807, %r5, %r849;
	// end inline asm
	cvt.u64.u32 	%rd784, %r845;
	shl.b64 	%rd785, %rd784, 32;
	cvt.u64.u32 	%rd786, %r844;
	or.b64  	%rd1077, %rd785, %rd786;
	// begin inline asm
	add.cc.u32 %r851, %r817, %r854;
	madc.lo.u32 %r852, %r818, %r5, %r856;
	// end inline asm
	cvt.u64.u32 	%rd787, %r852;
	shl.b64 	%rd788, %rd787, 32;
	cvt.u64.u32 	%rd789, %r851;
	or.b64  	%rd1076, %rd788, %rd789;
	// begin inline asm
	add.cc.u32 %r858, %r828, %r861;
	madc.lo.u32 %r859, %r829, %r5, %r863;
	// end inline asm
	cvt.u64.u32 	%rd790, %r859;
	shl.b64 	%rd791, %rd790, 32;
	cvt.u64.u32 	%rd792, %r858;
	or.b64  	%rd1075, %rd791, %rd792;
	prmt.b32 	%r901, %r838, %r845, %r894;
	prmt.b32 	%r868, %r837, %r901, %r896;
	prmt.b32 	%r870, %r845, %r837, %r897;
	prmt.b32 	%r875, %r844, %r901, %r898;
	prmt.b32 	%r877, %r844, %r838, %r899;
	prmt.b32 	%r902, %r852, %r859, %r894;
	prmt.b32 	%r882, %r851, %r902, %r896;
	prmt.b32 	%r884, %r859, %r851, %r897;
	prmt.b32 	%r889, %r858, %r902, %r898;
	prmt.b32 	%r891, %r858, %r852, %r899;
	// begin inline asm
	add.cc.u32 %r865, %r867, %r868;
	madc.lo.u32 %r866, %r869, %r5, %r870;
	// end inline asm
	cvt.u64.u32 	%rd793, %r866;
	shl.b64 	%rd794, %rd793, 32;
	cvt.u64.u32 	%rd795, %r865;
	or.b64  	%rd1128, %rd794, %rd795;
	// begin inline asm
	add.cc.u32 %r872, %r874, %r875;
	madc.lo.u32 %r873, %r876, %r5, %r877;
	// end inline asm
	cvt.u64.u32 	%rd796, %r873;
	shl.b64 	%rd797, %rd796, 32;
	cvt.u64.u32 	%rd798, %r872;
	or.b64  	%rd1073, %rd797, %rd798;
	// begin inline asm
	add.cc.u32 %r879, %r881, %r882;
	madc.lo.u32 %r880, %r883, %r5, %r884;
	// end inline asm
	cvt.u64.u32 	%rd799, %r880;
	shl.b64 	%rd800, %rd799, 32;
	cvt.u64.u32 	%rd801, %r879;
	or.b64  	%rd1072, %rd800, %rd801;
	// begin inline asm
	add.cc.u32 %r886, %r888, %r889;
	madc.lo.u32 %r887, %r890, %r5, %r891;
	// end inline asm
	cvt.u64.u32 	%rd802, %r887;
	shl.b64 	%rd803, %rd802, 32;
	cvt.u64.u32 	%rd804, %r886;
	or.b64  	%rd1071, %rd803, %rd804;
	add.s32 	%r116, %r1421, -1;
	setp.gt.u32 	%p38, %r1421, 3;
	mov.b32 	%r1422, 2;
	mov.u32 	%r1421, %r116;
	@%p38 bra 	$L__BB3_38;
$L__BB3_39:
	setp.ne.s32 	%p39, %r1422, 2;
	@%p39 bra 	$L__BB3_41;
	shl.b64 	%rd809, %rd1076, 32;
	shr.u64 	%rd810, %rd1076, 32;
